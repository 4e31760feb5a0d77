// Kernel parameter blocks and launchers (kernels.cu), used by abi.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "lp_internal.h"

namespace lpb {

constexpr int kThreads = 1024;          // persistent kernels: 32 warps per CTA
// Register-streaming full θ-pass CTA size.  (512 threads with twice the loads in flight
// per thread measured no faster on C4 and slower on C3.)
constexpr int kFullThreads = 1024;
constexpr int kMaxSmemBytes = 200 * 1024;
constexpr int kCpSmemBytes = 226 * 1024;    // compact stable kernels (+ ~50 B static <= 227 KB)
constexpr int kKeySmemBytes = 208 * 1024;   // key-space summary (register-streaming kernel only)
constexpr int kMaxRuns = 256;          // key mode: bucket runs of the row order kept in shared
                                       // memory (more: LEAD passes stream every octet)

// Run status bit flags (LMParams / STParams status_out).  Sticky: a queue overflow is
// never masked by a later cap or guard; the host checks kStOverflow first.
constexpr int kStGuard = 1;     // pass guard (n_ext + 2 passes) hit
constexpr int kStOverflow = 2;  // a candidate queue overflowed (internal error)
constexpr int kStCapped = 4;    // stopped at lp_run.max_passes before the fixpoint
constexpr int kSmemLimit = 232448 - 1024;  // opt-in smem per CTA on sm_100 minus static
constexpr int kMaxSmemSegs = 64;       // segment table copied to shared memory up to this size
constexpr int kSmemQueue = 768;        // candidate queue entries kept in shared memory per CTA
#ifndef LP_STREAM_WARPS
#define LP_STREAM_WARPS 28
#endif
constexpr int kStreamWarps = LP_STREAM_WARPS;
constexpr int kBucketWords = 256;
constexpr int kStQueue = 2048;         // stable search: candidate rows queued per CTA and pass
constexpr int kStQueueA = 1024;        // ... (record, lead) pairs in armed passes

// Least-model fixpoint (full θ-pass and frontier variants).
struct LMParams {
    const Segment *segs;
    int32_t nseg;
    int32_t n;                 // atoms of the encoded program (originals + P^δ auxiliaries)
    int32_t n_out;             // original atoms: v0, model and stage range
    int32_t n_ext_atoms;       // extended atoms (bounds checks)
    int32_t n_order_cap;       // entries of the derivation list (bounds checks)
    const int32_t *col;
    const int32_t *head;
    uint32_t *buf0;            // truth vector v_k (bit a of word a>>5); double buffer
    uint32_t *buf1;
    int32_t nwords;            // 32-bit words per truth buffer
    // v_0 inputs (the prologue builds v_0 inside the persistent kernel)
    const uint32_t *v0;        // optional user start set, 32-bit view of the ABI words
    int32_t v0_words;          // 32-bit words of v0
    const uint32_t *factbits;  // [nwords] bit vector of the atoms with a fact rule
    // v0 == NULL: v_0 precomputed at load (facts | ⊤ words, the facts in id order, keys)
    const uint32_t *init_bits;
    const int32_t *init_list;
    const int32_t *init_klist; // (key mode)
    const uint32_t *init_ksum; // (key mode) v_0's key summary [ksm_words] + bucket mask [kBucketWords]
    int32_t n_init;
    int32_t top;               // ⊤
    unsigned long long *model_out;  // [out_wn] written by the epilogue: model words out_w0..
    int32_t model_split;       // 1 (page-locked host model buffer): the prologue writes v_0's words
                               //   (over PCIe, in the background of the passes), the epilogue
                               //   only the words that hold derived atoms
    int64_t out_w0, out_wn;
    int32_t *tail_next;        // the other-parity run counters, zeroed for the next call
    int32_t *status_next;
    // shared-memory copy of the truth vector: exact (shift 0) or a summary whose bit g
    // is the OR of atoms [g << shift, (g+1) << shift)
    uint32_t *summary;         // initial summary (global, built by the prologue)
    int32_t sm_words;
    int32_t shift;
    // derivation order list: initial atoms at [0, n0), then every atom in the pass /
    // level it became true; tail = next free slot (device counter)
    int32_t *order;
    int32_t *tail;
    int32_t *stage;            // optional [n]
    int32_t *pops;             // optional [pop_cap]
    int32_t pop_cap;
    int32_t *iters_out;
    int32_t *status_out;       // run status, bit flags kSt* (0 = converged, nothing dropped)
    int32_t *status_user;      // optional (lp_run.status_out, device): the final status word,
                               //   written by the epilogue
    int32_t max_passes;        // guard (n_ext + 2)
    int32_t user_cap;          // lp_run.max_passes (0 = to the fixpoint)
    // frontier variant
    const int64_t *occ_ptr;
    const int32_t *occ_slot;   // [4 * nnz]: (slot, head(slot), occ range of that head) per occurrence
    int32_t *fq;               // [2][n_order_cap][4] frontier level queues (atom, occ range), -1 = empty
    uint32_t *cnt;             // per-slot remaining-body counters
    int32_t cnt_bits;          // 4: nibbles, 8 per word; 8: bytes, 4 per word; 32: uint32
    unsigned long long *dbg;   // optional profiling timestamps (lpdbg_set_timing)
    int32_t dbg_clock;         // ... as SM clock64 values instead of %globaltimer (lpdbg_set_clock)
    // FILTER mode: per-CTA candidate queues (rows that passed the summary test)
    int32_t *qbuf;             // [grid][qcap]
    int32_t qcap;
    // full θ-pass schedule: LEAD passes stream only the lead
    // atom of every row (+ the head row when the truth test is exact) and verify the
    // survivors from a queue; STREAM passes stream every body position.
    int32_t pass_mode;         // 0 auto (LEAD until a pass queues > n_slots/dense_div
                               //   rows, STREAM from then on), 1 always LEAD, 2 always STREAM
    int32_t dense_div;
    int32_t predict;           // auto schedule: estimate the first LEAD pass (LP_NO_PREDICT: off)
    int64_t n_slots;
    int32_t *cand;             // [3] rows queued per pass (slot k % 3)
    unsigned long long *vent;  // [3] body entries the verification loaded per pass (k % 3)
    long long stream_entries;  // body entries (incl. padding) one STREAM pass reads
    int32_t auto_stream_first; // auto schedule starts with STREAM passes (long bodies)
    // small-program kernel (lm_small_kernel): rows as a blob of uint16 -- row records (nr x 4:
    // head, body begin, body end, first body atom or 0xFFFF) | body (nnz) | occ_ptr
    // (n_ext + 1) | occ row (nnz), fact heads and always-true body atoms dropped
    const uint4 *sm_blob;
    int32_t sm_blob16, sm_nr, sm_nnz;
    int32_t stage_planes;      // cluster kernel: lead / head / col planes copied to shared memory
    int32_t cl_threads;        // cluster kernel: threads per CTA (0: kThreads)
    int32_t fr_cl_threads;     // one-cluster frontier launches: threads per CTA (0: kThreads)
    int32_t overlap;           // LEAD passes verify while they stream (warp-specialised)
    long long overlap_min_bytes;  // ... when the pass streams at least this many bytes
    // pipelined key-mode LEAD passes (lm_pipe): rows by lead atom, and the counter of the
    // split grid barrier; locc_ptr == NULL = not pipelined
    const int32_t *locc_ptr;   // [n_ext + 1]
    const int32_t *locc_slot;  // [rows]: the slots whose body position 0 is atom a
    uint32_t *pbar;
    unsigned long long *lbar;  // [2] (armed kernel) the pass barrier words, by pass parity
    int32_t *pcnt;             // [3] atoms appended to the derivation list per pass (slot
                               //     k % 3): read by every CTA after the pass's barrier,
                               //     never written again before the next one
    unsigned long long *stats; // [4] algorithmic bytes, LEAD passes, rows verified,
                               //     body entries loaded by verification
    long long lead_bytes;      // bytes one LEAD / STREAM pass streams (program planes only)
    long long stream_bytes;
    // summary mode key plane: LEAD passes stream the key group of
    // the lead atom (8 bits + a per-octet bucket) and test it against a summary in key space, where the
    // atoms that can become true (heads, facts) get fine groups and the rest share
    // coarse ones.  STREAM passes switch the shared copy back to the atom-id summary.
    const void *lead_codes;    // [n_slots] low key_bits bits of the lead atom's key group
                               //   (uint16 or uint8), or NULL (no key mode)
    const void *octet_tag;     // [n_slots / 8] bucket (group >> key_bits) | padding << 5 (uint8,
                               //   16-bit codes) or << 13 (uint16, 8-bit codes)
    int32_t key_bits;          // 16 (default) or 8 (LP_LOAD_KEY8)
    const int32_t *lead32;     // exact mode: [n_slots] body position 0 of every slot (flat)
    // exact mode, armed LEAD passes: rows by lead atom (arm_ptr[a] .. arm_ptr[a+1]) as
    // records [2 x int4: (head, L, body 1, body 2), (body 3, body 4, body 5, slot)], and the
    // capacity of each of the two per-CTA lists (shared memory after the truth words)
    const int32_t *arm_ptr;
    const int4 *arec;          // NULL: LEAD passes stream the lead / head planes
    int32_t arm_cap;
    const uint16_t *xlead16;   // exact mode, ids < 2^21: low 16 bits of lead / head, and per
    const uint16_t *xhead16;   //   octet lead bucket | head bucket << 5 | padding << 10
    const uint16_t *xtag;
    // key mode: the rows of every segment are in runs of one lead bucket (encode.cpp
    // bucket_rows); a LEAD pass streams only the octets of runs whose bucket has a set
    // summary bit.  nruns == 0: no table, every octet streamed.
    const int4 *runs;          // [nruns] (first octet, octets, bucket, 0), in slot order
    int32_t nruns;
    const int32_t *key_of;     // [n_ext] key of every extended atom
    int32_t *korder;           // [n_ext + 1] key of order[i] (written with it)
    int32_t ksm_words;         // words of the key-space summary (shared memory)
    int32_t kshift;
    int32_t prefetch;          // L2 prefetch of what the next pass / level loads (LP_NO_PREFETCH: off)
};

// profiling hook (not part of the ABI): per-CTA %globaltimer stamps
void set_debug_timing(unsigned long long *buf);
unsigned long long *debug_timing();
void set_debug_clock(int on);
int debug_clock();

// Batched (bit-sliced) stable-model fixpoint.
struct STParams {
    const Segment *segs;
    int32_t nseg;
    int32_t n_ext;
    const int32_t *col;
    const int32_t *head;
    unsigned long long *T0;    // [n_ext][Wp] words, double buffer
    unsigned long long *T1;
    int32_t Wp;                // words per row (even)
    const uint32_t *any_init;  // bit g: some row of atoms [g<<any_shift, (g+1)<<any_shift)
    int32_t any_words;         //        is nonzero in T_0 (a superset filter)
    int32_t any_shift;
    int32_t *order;            // [3][ring_cap] rows changed in pass k: segment k % 3
    int32_t ring_cap;          // n_ext + 1 (a row is listed at most once per pass)
    int32_t *tail;
    int32_t *pcnt;             // [3] per-pass append counters (slot k % 3)
    uint32_t *gfull;           // [any_words] rows true in every guess (use_full only)
    int32_t use_full;          // exact any-filter with room for the full bits
    unsigned long long *dbg;   // optional [64][4]: barrier exit, candidate rows, last CTA's
                               //   pass-top done, last CTA's scan done (per pass)
    const int32_t *lead32;     // exact mode: flat lead plane (one scan loop), else NULL
    // armed passes: rows by lead atom (arm_ptr) as 32-byte records (as LMParams); CTA b owns
    // records [b * arm_cap, (b + 1) * arm_cap) (arec NULL: the scan)
    const int32_t *arm_ptr;
    const int4 *arec;
    int32_t arm_cap;
    unsigned long long *lbar;  // [2] the pass barrier words (grid launches), by pass parity
    int32_t cta_queue;         // candidates shared by the CTA's warps (slots < 2^27, <= 32 segments)
    int64_t n_slots;
    int32_t W;                 // guess words in use (the rest of Wp is padding)
    int64_t G;                 // guesses
    int32_t *mark;             // [n_ext] pass tag of the last push (0: row never changed)
    int32_t *passes_out;
    int32_t *status_out;       // bit flags kSt*
    int32_t *status_user;      // optional device copy of the final status (lp_run.status_out)
    int32_t max_passes;
    // the rest of the call, fused into the same cooperative launch (clear -> T_0 -> fixpoint
    // -> stability check, grid barriers in between)
    int32_t n_atoms;                    // n: row of b̄_j is n + j
    int32_t k;                          // negated atoms
    const int32_t *negated;             // [k] atom a_j (check: a_j ∈ LM ⟺ b̄_j = 0)
    const int32_t *negated_ext;         // [k] row of b̄_j
    const int32_t *free_rank;           // [k] bit of b̄_j in the binary-counting guess id, -1: forced 0
    const unsigned long long *guesses;  // [k][W] the caller's guesses, or NULL (binary counting)
    int64_t woff;                       // first guess word (guess_offset / 64)
    const int32_t *facts;               // [nfacts] rows all-ones in T_0 (with ⊤ = top)
    int32_t nfacts;
    int32_t top;
    uint32_t *any_rw;                   // = any_init, built by the T_0 phase
    int32_t clear_rows;                 // zero the rows the previous call changed (mark != 0)
    unsigned long long *accepted;       // [W] accepted-guess mask (check)
    long long *n_accepted;
    // guess-space reduction (st_search_kernel, lp_stable_search): the round's columns are
    // gbuf ([k][W], = guesses), rewritten in place by the local-search move
    unsigned long long *gbuf;
    unsigned long long seed;
    int32_t max_rounds;
    int32_t *rounds_out;
    int32_t *passes_sum_out;            // whole-matrix passes summed over the rounds
    // compact kernel (st_compact_kernel): the live
    // sub-program -- the rows that can fire in some guess, over the atoms A* that can be true
    // in some guess (the closure of the facts with every abar_j true, computed by lp_load)
    // -- as one blob of uint16: row records (nr x 4: head, body begin, body end, first body
    // atom -- 0xFFFF when the body is empty) | body (nnz) | occ_ptr
    // (na+1) | occ row (nnz) | init (na: -1 zero in T_0, j >= 0 abar_j) | the rows whose
    // (compact) body holds abar atoms only: all that can fire in pass 0 (n0).  Compact atoms
    // are A* minus the all-ones rows (⊤, the facts), whose compact id reads -2.
    const uint4 *cp_blob;
    int32_t cp_blob16;                  // its size in 16-byte units
    int32_t cp_na, cp_nr, cp_nnz, cp_n0;  // atoms of A*, live rows, their body entries, pass-0 rows
    const int32_t *cp_atom;             // [na] extended atom id of compact atom c
    const int32_t *cp_neg;              // [k] compact id of a_j (-1: not in A*, never true; -2: a fact)
    const int32_t *cp_abar;             // [k] compact id of abar_j
    unsigned long long *cp_C;           // uint32 [2W][na]: the fixpoint matrix over the compact atoms,
                                        //   one row per 32-column half-word
    int32_t *cp_pw;                     // [2W] passes of each half-word
    int32_t *cp_done;                   // CTAs finished (self-resetting; the last one reduces)
    int32_t *cp_rp;                     // [3] search: a round's passes (max over words), slot r % 3
};

// Multi-GPU exchange step (lp_shard_combine).
constexpr int kMaxRanks = 64;
struct ShardCombineParams {
    const unsigned long long *gathered;  // [world][stride]: owned words, status word last
    int32_t world;
    int64_t stride;
    int64_t word_lo[kMaxRanks];
    int64_t word_cnt[kMaxRanks];
    const unsigned long long *v;         // [n_words] v_k
    unsigned long long *v_next;          // [n_words] v_{k+1}
    int64_t n_words;
    int32_t *changed;                    // 1: some rank's pass derived an atom
    int32_t *pops;                       // optional: += |v_{k+1}|
};

// ---- launchers (return cudaError_t of the launch) -----------------------------------
cudaError_t launch_shard_combine(const ShardCombineParams &q, cudaStream_t st);
// Each least-model call is ONE cooperative launch: v_0 prologue, the fixpoint loop and
// the model extraction all run inside the persistent kernel.
cudaError_t launch_lm_full(const LMParams &p, bool exact, int blocks, size_t smem, cudaStream_t st);
// cluster > 0: ONE thread-block cluster of that many CTAs with cluster barriers between
// passes (small programs); else the cooperative grid
cudaError_t launch_lm_frontier(const LMParams &p, int blocks, cudaStream_t st, int cluster);
int cluster_size_for(int which, int want, size_t smem);
// Exact-mode programs small enough for one thread-block cluster (truth in shared memory,
// DSMEM exchange, cluster barriers): the whole fixpoint in one cluster launch.
cudaError_t launch_lm_cluster(const LMParams &p, int cluster, size_t smem, cudaStream_t st);
// Programs whose rows fit shared memory in 16-bit ids: ONE CTA, semi-naive row lists.
cudaError_t launch_lm_small(const LMParams &p, size_t smem, cudaStream_t st, int threads = 0);
int lm_cluster_max(int want, size_t smem);

// One cooperative launch per stable call: clear the previous call's rows, build T_0, the
// fixpoint loop, the stability check.
cudaError_t launch_st_fused(const STParams &p, int blocks, size_t smem, cudaStream_t st, int cluster);
// The same call on the live sub-program held in shared memory, a CTA per guess word (no
// grid barrier: an ordinary launch).
cudaError_t launch_st_compact(const STParams &p, int blocks, size_t smem, cudaStream_t st, int threads = 0);
// ... the guess-space search on it (cooperative: one grid barrier per round; gbuf holds two
// column buffers [2][k][W])
cudaError_t launch_st_search_compact(const STParams &p, int blocks, size_t smem, cudaStream_t st);
// ... and its compact matrix C scattered into the zeroed T0 (for the matrix / column readback)
cudaError_t launch_st_expand(const STParams &p, cudaStream_t st);
// Guess-space reduction: all rounds of sampling + local search in one cooperative launch.
cudaError_t launch_st_search(const STParams &p, int blocks, size_t smem, cudaStream_t st, int cluster);
cudaError_t launch_st_column(const STParams &p, int32_t n, int64_t g, unsigned long long *out,
                             cudaStream_t st);

// occupancy helpers
int lm_full_blocks_per_sm(bool exact, size_t smem);
int lm_frontier_blocks_per_sm();
int st_blocks_per_sm(size_t smem);
int st_compact_blocks_per_sm(int which, size_t smem);
cudaError_t prepare_kernels(size_t lm_smem, size_t st_smem);

}  // namespace lpb
