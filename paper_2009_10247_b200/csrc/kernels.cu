// sm_100a kernels of the least-model / stable-model hot path.
//
//   lm_init_*          v_0 = v0 ∪ facts ∪ {⊤}                         (row a3; Def. 4)
//   lm_full_kernel     persistent fused θ-pass loop: every AND-row's body is tested
//                      against the bit-packed truth vector, firing rows OR their head
//                      bit into v_{k+1}, the changed flag is the growth of the
//                      derivation list; one cooperative launch runs all passes to the
//                      fixpoint                               (rows a4, a5; Alg. 1)
//   lm_frontier_kernel level-synchronous semi-naive variant: only the rows whose
//                      bodies contain newly-true atoms are touched   (row a6)
//   st_fixpoint_kernel one cooperative launch per stable call: bit-sliced initial
//                      matrix, 64 guesses per word (row a7; Def. 8), the batched
//                      θ-pass loop over it (row a8; Alg. 2) and the complementarity
//                      test a_j + abar_j = 1 per guess (row a9; Alg. 3)
//
// See DESIGN.md for the layout, the roofline of each kernel and the readings of the
// paper they implement.
#include <cooperative_groups.h>

#include <type_traits>

#include "kernels.h"

namespace cg = cooperative_groups;

// Bounds checks of the derived indices (build with -DLP_CHECKS; tools/checked_build.sh):
// a failed check prints the site and traps, so the call fails with a CUDA error.
#ifdef LP_CHECKS
#include <cstdio>
#define LP_CHECK(cond)                                                                     \
    do {                                                                                   \
        if (!(cond)) {                                                                     \
            printf("LP_CHECK failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__);            \
            __trap();                                                                      \
        }                                                                                  \
    } while (0)
#else
#define LP_CHECK(cond) do { } while (0)
#endif

#ifndef LP_OCT_U
#define LP_OCT_U 8   // 8-bit key plane: octets in flight per thread (8 measured best)
#endif

namespace lpb {

// ------------------------------------------------------------------------------------
// memory helpers
// ------------------------------------------------------------------------------------

// Streaming 128-bit load of read-only program data: no L1 allocation (no reuse).
__device__ __forceinline__ int4 ld_stream(const int4 *p) {
    int4 r;
    asm("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
        : "l"(p));
    return r;
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// L2 prefetch (fire and forget): pulls a line that a later pass / level will load out of
// HBM while the grid waits at its barrier.
__device__ __forceinline__ void prefetch_l2(const void *ptr) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(ptr));
}

static unsigned long long *g_dbg = nullptr;
static int g_dbg_clock = 0;
void set_debug_timing(unsigned long long *buf) { g_dbg = buf; }
unsigned long long *debug_timing() { return g_dbg; }
void set_debug_clock(int on) { g_dbg_clock = on; }
int debug_clock() { return g_dbg_clock; }

// The barrier between passes: the whole cooperative grid, or -- for kernels launched as ONE
// thread-block cluster (small programs: DESIGN.md "Cluster launches") -- the cluster
// barrier (release / acquire at cluster scope, which orders the CTAs' global-memory
// accesses too).
template <bool CL>
__device__ __forceinline__ void pass_barrier() {
    if constexpr (CL) cg::this_cluster().sync();
    else cg::this_grid().sync();
}

// The per-pass counters every thread needs right after a grid barrier are loaded by ONE
// thread per CTA and broadcast through shared memory: the same address from every warp
// of the grid (~4.7 k requests) queues on one L2 slice for microseconds.
struct PassCounts {
    int32_t appended;           // pcnt[k % 3]
    int32_t queued;             // cand[k % 3]
    unsigned long long vent;    // vent[k % 3]
};

__device__ __forceinline__ PassCounts cta_pass_counts(const int32_t *pcnt, const int32_t *cand,
                                                      const unsigned long long *vent) {
    __shared__ PassCounts s;
    if (threadIdx.x == 0) {
        s.appended = __ldcg(pcnt);
        s.queued = cand ? __ldcg(cand) : 0;
        s.vent = vent ? __ldcg(vent) : 0ull;
    }
    __syncthreads();
    return s;   // (every call site reaches a grid barrier before the next call rewrites s)
}

__device__ __forceinline__ bool sm_bit(const uint32_t *sm, uint32_t x) {
    return (sm[x >> 5] >> (x & 31)) & 1u;
}

// ------------------------------------------------------------------------------------
// least model: initial vector
// ------------------------------------------------------------------------------------

// Copy nw (multiple of 4) 32-bit words global -> shared with 16-byte loads, 4 in flight.
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
        "r"(parity) : "memory");
}

__device__ __forceinline__ void bulk_g2s_plain(void *dst, const void *src, uint32_t bytes,
                                               uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ void smem_fill(uint32_t *sm, const uint32_t *src, int32_t nw) {
    const int4 *s4 = reinterpret_cast<const int4 *>(src);
    int4 *d4 = reinterpret_cast<int4 *>(sm);
    const int32_t n4 = nw >> 2;
    for (int32_t i0 = threadIdx.x; i0 < n4; i0 += 4 * blockDim.x) {
        int4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int32_t i = i0 + u * blockDim.x;
            v[u] = i < n4 ? __ldcg(s4 + i) : make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int32_t i = i0 + u * blockDim.x;
            if (i < n4) d4[i] = v[u];
        }
    }
}

// Does the full θ-pass start with LEAD passes (else STREAM passes, which need the atom-id
// summary of v_0 in summary mode)?
__device__ __forceinline__ bool starts_lead(const LMParams &p) {
    return p.pass_mode == 1 || (p.pass_mode == 0 && !p.auto_stream_first);
}

// Reserve `cnt` consecutive list slots for every thread of the CTA with ONE atomic (all
// threads of the block must call it; two barriers).
__device__ __forceinline__ int32_t block_reserve(int32_t *tail, int32_t cnt) {
    __shared__ int32_t wsum[33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
        int32_t run = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
            const int32_t t = wsum[i];
            wsum[i] = run;
            run += t;
        }
        wsum[32] = run ? atomicAdd(tail, run) : 0;
    }
    __syncthreads();
    const int32_t r = wsum[32] + wsum[warp] + incl - cnt;
    __syncthreads();   // (wsum is reused by the next call)
    return r;
}

constexpr int kSplitFencePass = 2;   // (see model_split in lm_full_kernel)

// Model word i (original atoms 64i .. 64i+63) from its two 32-bit truth words, into the
// output window (lp_run.out_word_lo / out_word_count).
__device__ __forceinline__ void model_word_out(const LMParams &p, int64_t i, uint32_t lo, uint32_t hi) {
    if (i < p.out_w0 || i >= p.out_w0 + p.out_wn) return;
    unsigned long long v = (unsigned long long)lo | ((unsigned long long)hi << 32);
    const int64_t a0 = i * 64;
    if (a0 + 64 > p.n_out) v &= a0 >= p.n_out ? 0ull : (1ull << (uint32_t)(p.n_out - a0)) - 1ull;
    p.model_out[i - p.out_w0] = v;
}

// In-kernel prologue of every least-model kernel (no separate init launches):
//   v_0 word w = (v0[w] restricted to original atoms) | facts[w] | ⊤,
// written to both buffers.  Warps walk consecutive truth words (coalesced); each lane
// lists the original atoms of its word into the derivation list (slots reserved once
// per warp), writes their stages (0, or -1 for false atoms; one coalesced row per word
// of the warp) and, in summary mode, lists the atoms' keys (LEAD passes: every CTA builds
// its key-space summary from that list) and/or adds the word to the atom-id summary
// (STREAM passes, zero on entry).
// Also zeroes the other-parity run counters for the next call.
__device__ __noinline__ void lm_prologue(const LMParams &p, bool summary_mode, int64_t gtid,
                                         int64_t gthreads) {
    if (gtid == 0) {
        *p.tail_next = 0;
        *p.status_next = 0;
        p.pcnt[0] = p.pcnt[1] = p.pcnt[2] = 0;
        if (p.pbar) *p.pbar = 0u;
        if (p.lbar) p.lbar[0] = p.lbar[1] = 0ull;   // (read after the prologue's grid barrier)
    }
    const bool keys = summary_mode && p.lead_codes;
    const bool osum = summary_mode && !(keys && starts_lead(p));
    if (!p.v0 && !osum && p.init_list) {
        // v0 = facts only: the initial words and list were built at load, so
        // this is a plain copy -- no per-warp reservations on the list tail
        const int4 *ib = reinterpret_cast<const int4 *>(p.init_bits);
        int4 *b0 = reinterpret_cast<int4 *>(p.buf0);
        int4 *b1 = reinterpret_cast<int4 *>(p.buf1);
        for (int64_t w = gtid; w < (p.nwords >> 2); w += gthreads) {
            const int4 v = __ldg(ib + w);
            b0[w] = v;
            b1[w] = v;
            if (p.model_split) {   // model words 2w, 2w+1 (original atoms only)
                model_word_out(p, 2 * w, (uint32_t)v.x, (uint32_t)v.y);
                model_word_out(p, 2 * w + 1, (uint32_t)v.z, (uint32_t)v.w);
            }
        }
        // (split model output: the system fence that orders these stores before the
        // epilogue's comes passes later, see lm_full_kernel -- by then they are done)
        for (int64_t i = gtid; i < p.n_init; i += gthreads) {
            p.order[i] = __ldg(p.init_list + i);
            if (keys) p.korder[i] = __ldg(p.init_klist + i);
        }
        if (p.stage)
            for (int64_t a = gtid; a < p.n_out; a += gthreads)
                p.stage[a] = ((__ldg(p.init_bits + (a >> 5)) >> (a & 31)) & 1u) ? 0 : -1;
        if (gtid == 0) *p.tail = p.n_init;
        return;
    }
    const int lane = threadIdx.x & 31;
    // block-uniform loop: list slots are reserved once per CTA and iteration
    for (int64_t b0 = gtid - threadIdx.x; b0 < p.nwords; b0 += gthreads) {
        const int64_t w0 = b0 + (threadIdx.x & ~31);
        const int64_t w = b0 + threadIdx.x;
        const int64_t lo = w * 32;
        uint32_t orig = 0, bits = 0;
        if (w < p.nwords) {
            orig = __ldg(p.factbits + w);
            uint32_t v = (p.v0 && w < p.v0_words) ? __ldg(p.v0 + w) : 0u;   // originals only
            if (lo + 32 > p.n_out) v &= lo >= p.n_out ? 0u : ((1u << (uint32_t)(p.n_out - lo)) - 1u);
            orig |= v;
            if (lo + 32 > p.n) orig &= lo >= p.n ? 0u : ((1u << (uint32_t)(p.n - lo)) - 1u);
            bits = orig;
            if (w == (p.top >> 5)) bits |= 1u << (p.top & 31);
            p.buf0[w] = bits;
            p.buf1[w] = bits;
        }
        if (p.model_split) {   // model word w/2 from this lane's and the next lane's originals
            const uint32_t hi = __shfl_down_sync(0xFFFFFFFFu, orig, 1);
            if (!(w & 1) && w < p.nwords) model_word_out(p, w >> 1, orig, (w + 1) < p.nwords ? hi : 0u);
        }
        int32_t pos = block_reserve(p.tail, __popc(orig));
        for (uint32_t b = orig; b;) {
            const int i = __ffs(b) - 1;
            b &= b - 1;
            LP_CHECK(pos >= 0 && pos < p.n_order_cap);
            if (keys) p.korder[pos] = __ldg(p.key_of + lo + i);   // the CTAs build their
                                                                // key summaries from it
            p.order[pos++] = (int32_t)(lo + i);
        }
        if (p.stage) {   // row i of the warp's 32x32 block = word w0+i, lane = bit
            for (int i = 0; i < 32; ++i) {
                const uint32_t oi = __shfl_sync(0xFFFFFFFFu, orig, i);
                const int64_t a = (w0 + i) * 32 + lane;
                if (a < p.n_out) p.stage[a] = ((oi >> lane) & 1u) ? 0 : -1;
            }
        }
        if (osum) {   // word w contributes to atom-id summary word w >> shift
            uint32_t c = 0;
            if (bits) {
                if (p.shift >= 5) {
                    c = 1u << ((uint32_t)(w >> (p.shift - 5)) & 31u);
                } else {
                    const int gs = 1 << p.shift;
                    const uint32_t gm = (1u << gs) - 1u;
                    for (int i = 0; i < 32 / gs; ++i)
                        if ((bits >> (i * gs)) & gm) c |= 1u << ((uint32_t)((lo >> p.shift) + i) & 31u);
                }
            }
            const int span = p.shift >= 5 ? 32 : (1 << p.shift);   // lanes per summary word
            for (int o = 1; o < span; o <<= 1) c |= __shfl_xor_sync(0xFFFFFFFFu, c, o);
            if ((lane & (span - 1)) == 0 && c) atomicOr(p.summary + (w >> p.shift), c);
        }
    }
}

// The summaries are zero on entry to the next call (the prologue ORs into them).
__device__ __forceinline__ void lm_zero_summaries(const LMParams &p, bool summary_mode, int64_t gtid,
                                                  int64_t gthreads) {
    if (!summary_mode) return;
    if (!(p.lead_codes && starts_lead(p)))
        for (int64_t w = gtid; w < p.sm_words; w += gthreads) p.summary[w] = 0u;
}

// In-kernel epilogue: the model over the original atoms, LSB-first uint64 words.
// `v` = the buffer the last pass wrote (v_{k+1}: complete after its barrier; at a
// fixpoint both buffers hold the model, after a capped pass only this one does).
__device__ __noinline__ void lm_extract(const LMParams &p, int64_t gtid, int64_t gthreads,
                                        const uint32_t *v_last, int32_t d0 = 0, int32_t d1 = -1) {
    // split mode (p.model_split, derivation list [d0, d1) given): the prologue wrote v_0's
    // words; only the words holding atoms derived since are written (a word written several
    // times gets the same final value each time)
    if (p.model_split && d1 >= d0) {
        for (int64_t i = d0 + gtid; i < d1; i += gthreads) {
            const int32_t a = __ldcg(p.order + i);
            if (a >= p.n_out) continue;
            const int64_t w = a >> 6;
            model_word_out(p, w, __ldcg(v_last + 2 * w), __ldcg(v_last + 2 * w + 1));
        }
        return;
    }
    // (lp_run.out_word_lo / out_word_count: only model words [w0, w0 + nw) are written,
    // to model_out[0 .. nw) -- a head-range shard's owned words)
    const int64_t nw = p.out_wn;
    for (int64_t i = gtid; i < nw; i += gthreads) {
        const int64_t w = p.out_w0 + i;
        unsigned long long v = (unsigned long long)__ldcg(v_last + 2 * w) |
                               ((unsigned long long)__ldcg(v_last + 2 * w + 1) << 32);
        const int64_t lo = w * 64;
        if (lo + 64 > p.n_out) v &= (1ull << (uint32_t)(p.n_out - lo)) - 1ull;
        p.model_out[i] = v;
    }
}

// ------------------------------------------------------------------------------------
// least model: fused θ-pass (full variant)
// ------------------------------------------------------------------------------------

struct PassCtx {
    const uint32_t *rd;  // v_k (global)
    uint32_t *wr;        // v_{k+1} (global)
    const uint32_t *sm;  // shared copy of v_k (EXACT) or of its summary
    int32_t *qbuf;       // this CTA's candidate queue (global, FILTER mode)
    int32_t *qcount;     // its fill counter (shared memory)
    int k;
    const uint32_t *bmask;  // key mode: bit b = some summary bit of bucket b is set (shared bitmap)
    const Segment *segs;    // the segment table (shared-memory copy when it fits)
    int32_t *sq;            // the first kSmemQueue queue entries (shared memory), or NULL
    int32_t *pc;            // this pass's append counter (p.pcnt[k % 3])
    int32_t base;           // derivation-list index of this pass's first append
    int32_t *sapp = nullptr;  // (armed kernel) this CTA's appends in the pass (shared memory):
                              // the level barrier carries their sum, so no count is read back
};

// Queue entry i of this CTA: shared memory for the first kSmemQueue entries (no global
// round trip for the usual few hundred survivors per pass), the global queue after that.
// (register-streaming kernel only; its PassCtx always has sq)
// An entry past both parts is dropped (the caller reports the overflow as status 2);
// shared-memory entries are always written, so a verifier waiting for one never hangs.
__device__ __forceinline__ void qput(const LMParams &p, const PassCtx &c, int32_t i, int32_t slot) {
    if (i < kSmemQueue) c.sq[i] = slot;
    else if (i - kSmemQueue < p.qcap) c.qbuf[i - kSmemQueue] = slot;
}

__device__ __forceinline__ int32_t qget(const PassCtx &c, int32_t i) {
    return i < kSmemQueue ? c.sq[i] : __ldcg(c.qbuf + (i - kSmemQueue));
}

// Smem test of 4 AND-rows at one body position; `fire` bit e = row e still alive.
template <bool EXACT>
__device__ __forceinline__ unsigned test4(int4 a, unsigned fire, const uint32_t *sm, int shift) {
    const uint32_t s = EXACT ? 0u : (uint32_t)shift;
    if ((fire & 1u) && !sm_bit(sm, (uint32_t)a.x >> s)) fire &= ~1u;
    if ((fire & 2u) && !sm_bit(sm, (uint32_t)a.y >> s)) fire &= ~2u;
    if ((fire & 4u) && !sm_bit(sm, (uint32_t)a.z >> s)) fire &= ~4u;
    if ((fire & 8u) && !sm_bit(sm, (uint32_t)a.w >> s)) fire &= ~8u;
    return fire;
}

// OR a firing row's head into v_{k+1}; the thread that sets a new bit appends the head
// to the derivation list (the pass's "changed" signal) and records its stage.
__device__ __forceinline__ void emit_head(const LMParams &p, const PassCtx &c, int32_t h,
                                          uint32_t cur_word, int32_t hkey = -1) {
    const uint32_t bit = 1u << (h & 31);
    if (cur_word & bit) return;                            // already in v_k
    const uint32_t old = atomicOr(c.wr + (h >> 5), bit);
    if (old & bit) return;                                 // another row set it this pass
    // one list reservation per group of converged lanes (the tail is one hot address)
    const unsigned m = __activemask();
    const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
    int32_t base = 0;
    if (lane == leader) {
        base = atomicAdd(c.pc, __popc(m));
        if (c.sapp) atomicAdd(c.sapp, __popc(m));
    }
    base = __shfl_sync(m, base, leader);
    const int32_t pos = c.base + base + __popc(m & ((1u << lane) - 1u));
    LP_CHECK(pos >= 0 && pos <= p.n_order_cap && h >= 0 && h < p.n_ext_atoms);
    p.order[pos] = h;
    // (armed passes look up h's arm range next pass: its arm_ptr line toward L2 now)
    if (p.prefetch && p.arec) prefetch_l2(p.arm_ptr + h);
    if (p.lead_codes) p.korder[pos] = hkey >= 0 ? hkey : __ldg(p.key_of + h);   // once per atom
    if (p.stage && h < p.n_out) p.stage[h] = c.k + 1;
}


// Exact test of one queued row against v_k: the shared copy when it is exact, else the
// truth vector in L2.  The head is looked at first -- a row whose head is already in
// v_k cannot change anything -- then body positions j0..L-1 (LEAD passes have already
// tested position 0 exactly in EXACT mode).  Returns the body entries it loaded.
template <bool EXACT>
__device__ __forceinline__ int verify_slot(const LMParams &p, const PassCtx &c, int32_t slot, int j0) {
    int lo = 0, hi = p.nseg - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (c.segs[mid].slot_off <= slot) lo = mid; else hi = mid - 1;
    }
    LP_CHECK(slot >= 0 && slot < p.n_slots);
    const int32_t L = c.segs[lo].L;
    const int64_t cp = c.segs[lo].count_pad;
    const int32_t *colp = p.col + c.segs[lo].col_off + (slot - c.segs[lo].slot_off);
    // the head and up to 8 body atoms are loaded together (one memory round trip),
    // then their truth words (a second one)
    constexpr int B = 8;
    uint32_t a[B], w[B];
    const int32_t h = __ldg(p.head + slot);
    const int n1 = min(B, L - j0);
#pragma unroll
    for (int j = 0; j < B; ++j) a[j] = j < n1 ? (uint32_t)__ldg(colp + (int64_t)(j0 + j) * cp) : 0u;
    const uint32_t hw = EXACT ? c.sm[h >> 5] : __ldcg(c.rd + (h >> 5));
    // (key mode: the head's key, loaded with the truth words -- the emit needs it for the
    // derivation list's key twin, and a load after the list reservation would add a round
    // trip before this thread reaches the barrier)
    const int32_t hkey = (!EXACT && p.lead_codes) ? __ldg(p.key_of + h) : -1;
#pragma unroll
    for (int j = 0; j < B; ++j)
        w[j] = j < n1 ? (EXACT ? c.sm[a[j] >> 5] : __ldcg(c.rd + (a[j] >> 5))) : ~0u;
    if ((hw >> (h & 31)) & 1u) return n1;     // head already in v_k: the row changes nothing
    bool ok = true;
#pragma unroll
    for (int j = 0; j < B; ++j) ok = ok && ((w[j] >> (a[j] & 31)) & 1u);
    int loaded = n1;
    for (int32_t jb = j0 + B; jb < L && ok; jb += 4) {   // bodies longer than 8
        uint32_t x[4], y[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) x[j] = jb + j < L ? (uint32_t)__ldg(colp + (int64_t)(jb + j) * cp) : 0u;
#pragma unroll
        for (int j = 0; j < 4; ++j)
            y[j] = jb + j < L ? (EXACT ? c.sm[x[j] >> 5] : __ldcg(c.rd + (x[j] >> 5))) : ~0u;
#pragma unroll
        for (int j = 0; j < 4; ++j) ok = ok && ((y[j] >> (x[j] & 31)) & 1u);
        loaded += min(4, L - jb);
    }
    if (ok) emit_head(p, c, h, hw, hkey);
    return loaded;
}

// Armed LEAD pass (exact mode): test one armed row -- its lead atom is in v_k -- against
// v_k in shared memory from its 32-byte record (head, L, body positions 1..5, slot; longer
// bodies read positions 6.. from the column planes).  A firing row's head is emitted.
// Returns true if the row stays armed (head not in v_{k+1}: some body atom is still false).
template <bool EXACT>
__device__ __forceinline__ bool armed_verify(const LMParams &p, const PassCtx &c, int32_t o, int &loaded) {
    const int4 r0 = __ldg(p.arec + 2 * (int64_t)o);
    const int4 r1 = __ldg(p.arec + 2 * (int64_t)o + 1);
    const int32_t h = r0.x, L = r0.y;
    LP_CHECK(h >= 0 && h < p.n_ext_atoms && L >= 1);
    const int32_t b[5] = {r0.z, r0.w, r1.x, r1.y, r1.z};
    bool ok = true;
    uint32_t hw;
    if (EXACT) {   // v_k in shared memory
        hw = c.sm[h >> 5];
#pragma unroll
        for (int j = 0; j < 5; ++j) ok = ok && (j + 1 >= L || sm_bit(c.sm, (uint32_t)b[j]));
    } else {       // v_k in L2: the head's and the body atoms' words in one round trip
        uint32_t w[5];
        hw = __ldcg(c.rd + (h >> 5));
#pragma unroll
        for (int j = 0; j < 5; ++j) w[j] = j + 1 < L ? __ldcg(c.rd + (b[j] >> 5)) : ~0u;
#pragma unroll
        for (int j = 0; j < 5; ++j) ok = ok && ((w[j] >> (b[j] & 31)) & 1u);
    }
    if ((hw >> (h & 31)) & 1u) return false;   // head in v_k: the row adds nothing, now or later
    loaded += min(L, 6) - 1;
    if (ok && L > 6) {   // positions 6.. of the row's segment
        const int32_t slot = r1.w;
        int lo = 0, hi = p.nseg - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (c.segs[mid].slot_off <= slot) lo = mid; else hi = mid - 1;
        }
        const int64_t cp = c.segs[lo].count_pad;
        const int32_t *colp = p.col + c.segs[lo].col_off + (slot - c.segs[lo].slot_off);
        for (int32_t j = 6; j < L && ok; ++j) {
            const uint32_t x = (uint32_t)__ldg(colp + (int64_t)j * cp);
            ok = EXACT ? sm_bit(c.sm, x) : ((__ldcg(c.rd + (x >> 5)) >> (x & 31)) & 1u);
        }
        loaded += L - 6;
    }
    if (!ok) return true;
    emit_head(p, c, h, hw);
    return false;
}

// FILTER mode: rows that passed the summary test are queued and verified in the
// pass epilogue with many independent L2 requests in flight, so the streaming loop
// never waits on a dependent L2 round trip.
// (The host sizes qcap so that a CTA's queue can hold every row it streams in a pass;
// an overflow is impossible by construction and would be reported as status 2.)
__device__ __forceinline__ void enqueue(const LMParams &p, const PassCtx &c, int32_t slot0,
                                        unsigned fire) {
    int32_t pos = atomicAdd(c.qcount, __popc(fire));
    if (pos + __popc(fire) > p.qcap + kSmemQueue) atomicOr(p.status_out, kStOverflow);
#pragma unroll
    for (int e = 0; e < 4; ++e)
        if ((fire >> e) & 1u) qput(p, c, pos++, slot0 + e);
}

// EXACT mode: the shared-memory test is exact, so a passing row fires; its head comes
// from the head row streamed together with the body positions (no dependent load).
__device__ __forceinline__ void fire_exact4(const LMParams &p, const PassCtx &c, int4 h,
                                            unsigned fire) {
    if (fire & 1u) emit_head(p, c, h.x, c.sm[h.x >> 5]);
    if (fire & 2u) emit_head(p, c, h.y, c.sm[h.y >> 5]);
    if (fire & 4u) emit_head(p, c, h.z, c.sm[h.z >> 5]);
    if (fire & 8u) emit_head(p, c, h.w, c.sm[h.w >> 5]);
}

// One body-length segment, 4 AND-rows per thread per int4 load, U quads in flight.
// FILTER mode streams the L body rows (heads are read only for verified candidates);
// EXACT mode streams the head row as well.
template <int L, int U, bool EXACT>
__device__ __forceinline__ int seg_pass(const LMParams &p, const Segment &sg, const PassCtx &c,
                                        int32_t gtid, int32_t gthreads) {
    int loads = 0;
    const int32_t nq = (int32_t)(sg.count_pad >> 2);   // slots < 2^31 (checked at load)
    const int32_t slot0 = (int32_t)sg.slot_off;
    const int4 *base = reinterpret_cast<const int4 *>(p.col + sg.col_off);
    const int4 *hbase = reinterpret_cast<const int4 *>(p.head + sg.slot_off);
    for (int32_t q0 = gtid; q0 < nq; q0 += gthreads * U) {
        int4 v[U][L];
        int4 hv[EXACT ? U : 1];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t q = q0 + u * gthreads;
#pragma unroll
            for (int j = 0; j < L; ++j)
                v[u][j] = q < nq ? ld_stream(base + (int64_t)j * nq + q) : make_int4(0, 0, 0, 0);
            if (EXACT) hv[EXACT ? u : 0] = q < nq ? ld_stream(hbase + q) : make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t q = q0 + u * gthreads;
            if (q >= nq) break;
            loads += L + (EXACT ? 1 : 0);
            unsigned fire = 0xFu;
#pragma unroll
            for (int j = 0; j < L; ++j) fire = test4<EXACT>(v[u][j], fire, c.sm, p.shift);
            if (fire) {
                if (EXACT) fire_exact4(p, c, hv[EXACT ? u : 0], fire);
                else enqueue(p, c, slot0 + q * 4, fire);
            }
        }
    }
    return loads;
}

// Bodies longer than 8: positions in chunks of 8 independent loads, and a quad stops
// loading once its 4 rows are all dead (short-circuit AND; long bodies usually die early).
// Returns the int4 loads it issued (the bytes this STREAM pass really read).
template <bool EXACT>
__device__ int seg_pass_generic(const LMParams &p, const Segment &sg, const PassCtx &c,
                                int32_t gtid, int32_t gthreads) {
    const int32_t nq = (int32_t)(sg.count_pad >> 2);
    const int32_t slot0 = (int32_t)sg.slot_off;
    const int4 *base = reinterpret_cast<const int4 *>(p.col + sg.col_off);
    const int4 *hbase = reinterpret_cast<const int4 *>(p.head + sg.slot_off);
    int loads = 0;
    for (int32_t q = gtid; q < nq; q += gthreads) {
        const int4 hv = EXACT ? ld_stream(hbase + q) : make_int4(0, 0, 0, 0);
        loads += EXACT ? 1 : 0;
        unsigned fire = 0xFu;
        for (int32_t j0 = 0; j0 < sg.L && fire; j0 += 8) {
            int4 v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
                v[j] = j0 + j < sg.L ? ld_stream(base + (int64_t)(j0 + j) * nq + q) : make_int4(0, 0, 0, 0);
            loads += min(8, sg.L - j0);
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (j0 + j < sg.L) fire = test4<EXACT>(v[j], fire, c.sm, p.shift);
        }
        if (fire) {
            if (EXACT) fire_exact4(p, c, hv, fire);
            else enqueue(p, c, slot0 + q * 4, fire);
        }
    }
    return loads;
}

// LEAD pass over one segment: stream only body position 0 (the lead atom, chosen at
// load time, encode.cpp) of 4 rows per int4 load, U quads in flight; EXACT mode also
// streams the head row and drops rows whose head is already in v_k.  Rows that survive
// go to this CTA's queue and are verified in the pass epilogue (verify_slot), so the
// other body positions are loaded only for the few rows whose lead atom is true.
template <int U, bool EXACT>
__device__ __forceinline__ void seg_lead(const LMParams &p, const Segment &sg, const PassCtx &c,
                                         int32_t gtid, int32_t gthreads) {
    const int32_t nq = (int32_t)(sg.count_pad >> 2);
    const int32_t slot0 = (int32_t)sg.slot_off;
    const int shift = p.shift;
    const int4 *base = reinterpret_cast<const int4 *>(p.col + sg.col_off);
    const int4 *hbase = reinterpret_cast<const int4 *>(p.head + sg.slot_off);
    for (int32_t q0 = gtid; q0 < nq; q0 += gthreads * U) {
        int4 v[U];
        int4 hv[EXACT ? U : 1];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t q = q0 + u * gthreads;
            v[u] = q < nq ? ld_stream(base + q) : make_int4(0, 0, 0, 0);
            if (EXACT) hv[EXACT ? u : 0] = q < nq ? ld_stream(hbase + q) : make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t q = q0 + u * gthreads;
            if (q >= nq) break;
            unsigned fire = test4<EXACT>(v[u], 0xFu, c.sm, shift);
            if (EXACT && fire) {   // keep the rows whose head is not yet in v_k
                const int4 h = hv[EXACT ? u : 0];
                fire &= (sm_bit(c.sm, (uint32_t)h.x) ? 0u : 1u) | (sm_bit(c.sm, (uint32_t)h.y) ? 0u : 2u) |
                        (sm_bit(c.sm, (uint32_t)h.z) ? 0u : 4u) | (sm_bit(c.sm, (uint32_t)h.w) ? 0u : 8u);
            }
            if (fire) enqueue(p, c, slot0 + q * 4, fire);
        }
    }
}

// LEAD pass in key mode: stream the key plane, 8 rows (one octet) per load of their
// codes plus the octet's tag (bucket = key group >> key_bits, and the number of trailing
// padding rows), U octets in flight per thread.  Row i is alive iff summary bit
// (bucket << key_bits | code[i]) is set; an octet whose bucket has no set bit is dead
// without a lookup.  Thread t takes octets t, t + gthreads, ...
__device__ __forceinline__ uint2 ld_stream8(const uint2 *p) {
    uint2 r;
    asm("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
}

__device__ __forceinline__ bool bucket_any(const uint32_t *bm, uint32_t b) {
    return (bm[b >> 5] >> (b & 31)) & 1u;
}

// KB = bits of the key group each row carries (16: uint16 codes, uint8 tags with 5 bucket
// bits; 8: uint8 codes, uint16 tags with 13 bucket bits); the octet's bucket is
// group >> KB and the tag's top 3 bits count its trailing padding rows.
template <int KB>
struct OctT {
    using vec = typename std::conditional<KB == 16, int4, uint2>::type;   // 8 codes
    using tag = typename std::conditional<KB == 16, uint8_t, uint16_t>::type;
    static constexpr uint32_t bmask = KB == 16 ? 31u : 0x1FFFu;
    static constexpr int pshift = KB == 16 ? 5 : 13;
    static __device__ __forceinline__ vec load(const vec *p) {
        if constexpr (KB == 16) return ld_stream(p);
        else return ld_stream8(p);
    }
    static __device__ __forceinline__ uint32_t code(const vec &v, int e) {   // row e of 8
        if constexpr (KB == 16) {
            const uint32_t w = e < 2 ? (uint32_t)v.x : e < 4 ? (uint32_t)v.y : e < 6 ? (uint32_t)v.z : (uint32_t)v.w;
            return (e & 1) ? (w >> 16) : (w & 0xFFFFu);
        } else {
            const uint32_t w = e < 4 ? v.x : v.y;
            return (w >> (8 * (e & 3))) & 0xFFu;
        }
    }
};

// Live runs.  The rows of each segment lie in runs of one lead
// bucket, and a run whose bucket has no set summary bit cannot hold a candidate -- so a
// key-mode LEAD pass streams only the octets of the live runs, never loading the others'
// codes.  Each CTA lists them in shared memory at the pass top (one warp, from the run
// table copied in at launch): beg[r] = first octet of live run r, pre[r] = live octets
// before it, pre[m] = total.  The stream deals VIRTUAL octet indices 0..total-1 over its
// threads and maps them through the list with a forward-only cursor (a thread's
// indices only grow).  With no table the list is the single range [0, n_slots / 8).
struct LiveList {
    const int32_t *beg;
    const int32_t *pre;
    int32_t total;
};

__device__ __forceinline__ bool bucket_any(const uint32_t *bm, uint32_t b);

// warp 0 of the CTA; the caller synchronises the CTA afterwards
__device__ __forceinline__ void build_live(const LMParams &p, const uint32_t *bmask, const int4 *runs_sm,
                                           int32_t *beg, int32_t *pre, int32_t *total) {
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    if (p.nruns == 0) {
        if (lane == 0) {
            beg[0] = 0;
            pre[0] = 0;
            pre[1] = (int32_t)(p.n_slots >> 3);
            *total = (int32_t)(p.n_slots >> 3);
        }
        return;
    }
    int32_t m = 0, tot = 0;
    for (int32_t i0 = 0; i0 < p.nruns; i0 += 32) {
        const int32_t i = i0 + lane;
        int4 r = make_int4(0, 0, 0, 0);
        bool live = false;
        if (i < p.nruns) {
            r = runs_sm[i];
            live = bucket_any(bmask, (uint32_t)r.z);
        }
        const int32_t len = live ? r.y : 0;
        int32_t inc = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
            if (lane >= o) inc += y;
        }
        const unsigned bal = __ballot_sync(0xFFFFFFFFu, live);
        if (live) {
            const int32_t k = m + __popc(bal & ((1u << lane) - 1u));
            beg[k] = r.x;
            pre[k] = tot + inc - len;
        }
        m += __popc(bal);
        tot += __shfl_sync(0xFFFFFFFFu, inc, 31);
    }
    if (lane == 0) {
        pre[m] = tot;   // sentinel: the cursor never passes the last live run
        *total = tot;
    }
}

// Octet indices of virtual indices vq0 + u * gth (u = 0..U-1); -1 past the total.
template <int U>
__device__ __forceinline__ void live_octets(const LiveList &lv, int32_t vq0, int32_t gth, int32_t &cur,
                                            int32_t (&q)[U]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int32_t vq = vq0 + u * gth;
        if (vq < lv.total) {
            while (lv.pre[cur + 1] <= vq) ++cur;
            q[u] = lv.beg[cur] + (vq - lv.pre[cur]);
        } else {
            q[u] = -1;
        }
    }
}

template <int U, int KB>
__device__ __forceinline__ void oct_load(const LMParams &p, const int32_t (&q)[U],
                                         typename OctT<KB>::vec (&v)[U], uint32_t (&tag)[U]) {
    using T = OctT<KB>;
    const typename T::vec *base = reinterpret_cast<const typename T::vec *>(p.lead_codes);
    const typename T::tag *tb = reinterpret_cast<const typename T::tag *>(p.octet_tag);
#pragma unroll
    for (int u = 0; u < U; ++u) {
        if (q[u] >= 0) {
            v[u] = T::load(base + q[u]);
            tag[u] = (uint32_t)__ldg(tb + q[u]);
        } else {
            v[u] = typename T::vec{};
            tag[u] = 0u;
        }
    }
}

template <int U, int KB>
__device__ __forceinline__ void oct_test(const LMParams &p, const PassCtx &c, const int32_t (&qi)[U],
                                         const typename OctT<KB>::vec (&v)[U], const uint32_t (&tag)[U]) {
    using T = OctT<KB>;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int32_t q = qi[u];
        if (q < 0) break;
        const uint32_t b = tag[u] & T::bmask;
        if (!bucket_any(c.bmask, b)) continue;            // bucket with no true key
        const uint32_t hi = b << KB;
        unsigned fire = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) fire |= (unsigned)sm_bit(c.sm, hi | T::code(v[u], e)) << e;
        fire &= 0xFFu >> (tag[u] >> T::pshift);           // trailing padding rows
        if (fire) {
            int32_t pos = atomicAdd(c.qcount, __popc(fire));
            if (pos + __popc(fire) > p.qcap + kSmemQueue) atomicOr(p.status_out, kStOverflow);
            const int32_t s0 = q * 8;
            for (unsigned f = fire; f; f &= f - 1) qput(p, c, pos++, s0 + __ffs(f) - 1);
        }
    }
}

// (issuing the first loads before the pass-top delta update, so they overlap its
// latency, measured slower: they compete with the delta's loads and add spills)
template <int U, int KB>
__device__ __forceinline__ void octets_lead_kb(const LMParams &p, const PassCtx &c, const LiveList &lv,
                                               int64_t gtid, int64_t gthreads) {
    const int32_t gth = (int32_t)gthreads;
    int32_t cur = 0;
    for (int32_t q0 = (int32_t)gtid; q0 < lv.total; q0 += gth * U) {
        typename OctT<KB>::vec v[U];
        uint32_t tag[U];
        int32_t q[U];
        live_octets<U>(lv, q0, gth, cur, q);
        oct_load<U, KB>(p, q, v, tag);
        oct_test<U, KB>(p, c, q, v, tag);
    }
}

// (16-bit codes: 4 octets = 64 bytes in flight per thread; 8-bit codes: 8 octets)
__device__ __forceinline__ void octets_lead(const LMParams &p, const PassCtx &c, const LiveList &lv,
                                            int64_t gtid, int64_t gthreads) {
    if (p.key_bits == 8) octets_lead_kb<LP_OCT_U, 8>(p, c, lv, gtid, gthreads);
    else octets_lead_kb<4, 16>(p, c, lv, gtid, gthreads);
}

// LEAD pass in exact mode over the 16-bit planes: 8 rows per 16-byte load of each plane
// plus the octet's tag; a row is queued when its lead atom is in v_k and its head is not.
template <int U>
__device__ __forceinline__ void octets_exact16(const LMParams &p, const PassCtx &c, int64_t gtid,
                                               int64_t gthreads) {
    const int32_t no = (int32_t)(p.n_slots >> 3);
    const int32_t gth = (int32_t)gthreads;
    const int4 *lb = reinterpret_cast<const int4 *>(p.xlead16);
    const int4 *hb = reinterpret_cast<const int4 *>(p.xhead16);
    for (int32_t q0 = (int32_t)gtid; q0 < no; q0 += gth * U) {
        int4 lv[U], hv[U];
        uint32_t tag[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t q = q0 + u * gth;
            lv[u] = q < no ? ld_stream(lb + q) : make_int4(0, 0, 0, 0);
            hv[u] = q < no ? ld_stream(hb + q) : make_int4(0, 0, 0, 0);
            tag[u] = q < no ? (uint32_t)__ldg(p.xtag + q) : 0u;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t q = q0 + u * gth;
            if (q >= no) break;
            const uint32_t lhi = (tag[u] & 31u) << 16, hhi = ((tag[u] >> 5) & 31u) << 16;
            const uint32_t lw[4] = {(uint32_t)lv[u].x, (uint32_t)lv[u].y, (uint32_t)lv[u].z, (uint32_t)lv[u].w};
            const uint32_t hw[4] = {(uint32_t)hv[u].x, (uint32_t)hv[u].y, (uint32_t)hv[u].z, (uint32_t)hv[u].w};
            unsigned fire = 0;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                fire |= (unsigned)(sm_bit(c.sm, lhi | (lw[e] & 0xFFFFu)) && !sm_bit(c.sm, hhi | (hw[e] & 0xFFFFu))) << (2 * e);
                fire |= (unsigned)(sm_bit(c.sm, lhi | (lw[e] >> 16)) && !sm_bit(c.sm, hhi | (hw[e] >> 16))) << (2 * e + 1);
            }
            fire &= 0xFFu >> (tag[u] >> 10);                  // trailing padding rows
            if (fire) {
                int32_t pos = atomicAdd(c.qcount, __popc(fire));
                if (pos + __popc(fire) > p.qcap + kSmemQueue) atomicOr(p.status_out, kStOverflow);
                for (unsigned f = fire; f; f &= f - 1) qput(p, c, pos++, q * 8 + __ffs(f) - 1);
            }
        }
    }
}

// LEAD pass in exact mode over the flat lead plane: lead32[slot] = body position 0 of
// every slot, contiguous across segments like the head plane, so one loop over quads
// covers the whole program (no per-segment bookkeeping): 4 rows per int4 of each plane,
// U quads in flight; rows with a true lead atom and a false head are queued.
template <int U>
__device__ __forceinline__ void flat_lead_exact(const LMParams &p, const PassCtx &c, int64_t gtid,
                                                int64_t gthreads) {
    const int32_t nq = (int32_t)(p.n_slots >> 2);
    const int32_t gth = (int32_t)gthreads;
    const int4 *lb = reinterpret_cast<const int4 *>(p.lead32);
    const int4 *hb = reinterpret_cast<const int4 *>(p.head);
    for (int32_t q0 = (int32_t)gtid; q0 < nq; q0 += gth * U) {
        int4 v[U], hv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t q = q0 + u * gth;
            v[u] = q < nq ? ld_stream(lb + q) : make_int4(0, 0, 0, 0);
            hv[u] = q < nq ? ld_stream(hb + q) : make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t q = q0 + u * gth;
            if (q >= nq) break;
            unsigned fire = test4<true>(v[u], 0xFu, c.sm, 0);
            if (fire) {
                const int4 h = hv[u];
                fire &= (sm_bit(c.sm, (uint32_t)h.x) ? 0u : 1u) | (sm_bit(c.sm, (uint32_t)h.y) ? 0u : 2u) |
                        (sm_bit(c.sm, (uint32_t)h.z) ? 0u : 4u) | (sm_bit(c.sm, (uint32_t)h.w) ? 0u : 8u);
            }
            if (fire) enqueue(p, c, q * 4, fire);
        }
    }
}

// Segment s starts at the thread after the one that took the last quad of segment s-1,
// so short segments spread over the whole grid instead of piling onto the lowest ids.
template <bool EXACT, bool LEAD>
__device__ __forceinline__ int all_segments(const LMParams &p, const PassCtx &c, int64_t gtid,
                                            int64_t gthreads) {
    const int32_t gth = (int32_t)gthreads;
    int32_t off = 0;
    int loads = 0;
    for (int32_t s = 0; s < p.nseg; ++s) {
        const Segment sg = c.segs[s];
        const int32_t gt = (int32_t)gtid >= off ? (int32_t)gtid - off : (int32_t)gtid - off + gth;
        off = (int32_t)(((int64_t)off + (sg.count_pad >> 2)) % gth);
        const int32_t gthreads = gth;
        if (LEAD) {   // (used only without a flat lead plane, see the caller)
            seg_lead<EXACT ? 4 : 8, EXACT>(p, sg, c, gt, gthreads);
            continue;
        }
        // U quads in flight per thread: 4-8 int4 loads (EXACT also streams heads)
        switch (sg.L) {
            case 1: loads += seg_pass<1, 4, EXACT>(p, sg, c, gt, gthreads); break;
            case 2: loads += seg_pass<2, 2, EXACT>(p, sg, c, gt, gthreads); break;
            case 3: loads += seg_pass<3, EXACT ? 2 : 1, EXACT>(p, sg, c, gt, gthreads); break;
            case 4: loads += seg_pass<4, 1, EXACT>(p, sg, c, gt, gthreads); break;
            case 5: loads += seg_pass<5, 1, EXACT>(p, sg, c, gt, gthreads); break;
            case 6: loads += seg_pass<6, 1, EXACT>(p, sg, c, gt, gthreads); break;
            case 7: loads += seg_pass<7, 1, EXACT>(p, sg, c, gt, gthreads); break;
            case 8: loads += seg_pass<8, 1, EXACT>(p, sg, c, gt, gthreads); break;
            default: loads += seg_pass_generic<EXACT>(p, sg, c, gt, gthreads); break;
        }
    }
    return loads;
}

// Mark bucket bk in the shared bucket mask.  With 16-bit codes all buckets live in one
// word, so a delta of thousands of atoms would serialise on it: test first, the atomic
// only for a bit not yet set.
__shared__ int32_t s_bmask_changed;   // a bucket bit was set since the live list was built

__device__ __forceinline__ void set_bucket(uint32_t *bmask, uint32_t bk) {
    const uint32_t bit = 1u << (bk & 31);
    if (!(*(volatile uint32_t *)(bmask + (bk >> 5)) & bit)) {
        atomicOr(bmask + (bk >> 5), bit);
        s_bmask_changed = 1;
    }
}

// Add derivation-list entries [i0, i1) to a CTA's shared copy of v_k: exact bits
// (EXACT), key groups (keys: the list's korder twin) or atom-id groups; in key mode the
// per-bucket any-bit mask too.  4 independent list reads in flight per thread.
template <bool EXACT>
__device__ __forceinline__ void add_to_shared(const LMParams &p, uint32_t *sm, uint32_t *bmask,
                                              int32_t i_begin, int32_t i_end, bool keys) {
    for (int64_t i0 = i_begin + threadIdx.x; i0 < i_end; i0 += 4 * (int64_t)blockDim.x) {
        uint32_t a[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = i0 + u * (int64_t)blockDim.x;
            a[u] = i < i_end ? (uint32_t)__ldcg((keys ? p.korder : p.order) + i) : 0xFFFFFFFFu;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (a[u] == 0xFFFFFFFFu) continue;
            a[u] = EXACT ? a[u] : keys ? (a[u] >> p.kshift) : (a[u] >> p.shift);
            LP_CHECK((a[u] >> 5) < (uint32_t)(keys ? p.ksm_words : p.sm_words));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (a[u] != 0xFFFFFFFFu) {
                atomicOr(sm + (a[u] >> 5), 1u << (a[u] & 31));
                if (!EXACT && keys) {   // the group's bucket (group >> key_bits) now has a set bit
                    const uint32_t bk = a[u] >> p.key_bits;
                    set_bucket(bmask, bk);
                }
            }
    }
}

// ------------------------------------------------------------------------------------
// least model: pipelined key-space LEAD passes
// ------------------------------------------------------------------------------------
//
// A LEAD pass's stream only needs the key summary, and the rows it finds with the
// summary of v_k are the rows with a true lead atom in v_{k+1} minus those whose lead
// atom became true in pass k.  Those few are listed by the lead-occurrence lists
// (locc: rows by body position 0).  So pass k+1's stream, filtered by v_k, runs while
// pass k's candidates are verified, and the barrier that closes pass k waits behind it:
//
//   phase k (after the barrier of pass k-1 and the delta Δ_{k-1} folded into the summary
//   of v_k):  28 warps stream the lead plane against summary(v_k) -> queue S_{k+1};
//              4 warps verify S_k ∪ locc(Δ_{k-1}) against v_k (body ⊆ v_k, head emitted
//              into v_{k+1}), arrive at the split barrier of pass k and wait for it;
//   then Δ_k is folded into the summary (v_{k+1}) and phase k+1 starts.
//
// Candidates are tested exactly (verify_slot), so the result is θ(M v_k) as in the
// unpipelined pass; S_1 = S_0 (both are the rows passing summary(v_0)).  The stream of
// the phase whose pass turns out to be the last one is abandoned when its barrier
// opens.  Queues: two per CTA (384 shared-memory entries + qcap global each), S_j in
// half h(j) = (j + 1) & 1 for j >= 1, S_0 in half 0.
constexpr int kPipeSq = kSmemQueue / 2;

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t *a) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
    return v;
}

__device__ __forceinline__ int32_t pipe_qget(const int32_t *sq, const int32_t *gq, int32_t i) {
    return i < kPipeSq ? sq[i] : __ldcg(gq + (i - kPipeSq));
}

template <int U, int KB>
__device__ __forceinline__ void pipe_stream_kb(const LMParams &p, const uint32_t *sm, const uint32_t *bmask,
                                               const LiveList &lv, int32_t *sq, int32_t *gq, int32_t *qcnt,
                                               const volatile int32_t *abandon, int64_t gtid,
                                               int64_t gthreads) {
    using T = OctT<KB>;
    const int32_t gth = (int32_t)gthreads;
    int32_t cur = 0;
    for (int32_t q0 = (int32_t)gtid; q0 < lv.total; q0 += gth * U) {
        if (*abandon) break;
        typename T::vec v[U];
        uint32_t tag[U];
        int32_t qi[U];
        live_octets<U>(lv, q0, gth, cur, qi);
        oct_load<U, KB>(p, qi, v, tag);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t q = qi[u];
            if (q < 0) break;
            const uint32_t b = tag[u] & T::bmask;
            if (!bucket_any(bmask, b)) continue;
            const uint32_t hi = b << KB;
            unsigned fire = 0;
#pragma unroll
            for (int e = 0; e < 8; ++e) fire |= (unsigned)sm_bit(sm, hi | T::code(v[u], e)) << e;
            fire &= 0xFFu >> (tag[u] >> T::pshift);
            if (fire) {
                int32_t pos = atomicAdd(qcnt, __popc(fire));
                if (pos + __popc(fire) > p.qcap + kPipeSq) atomicOr(p.status_out, kStOverflow);
                const int32_t s0 = q * 8;
                for (unsigned f = fire; f; f &= f - 1, ++pos) {
                    if (pos < kPipeSq) sq[pos] = s0 + __ffs(f) - 1;
                    else if (pos - kPipeSq < p.qcap) gq[pos - kPipeSq] = s0 + __ffs(f) - 1;
                }
            }
        }
    }
}

__device__ __forceinline__ void pipe_stream(const LMParams &p, const uint32_t *sm, const uint32_t *bmask,
                                            const LiveList &lv, int32_t *sq, int32_t *gq, int32_t *qcnt,
                                            const volatile int32_t *abandon, int64_t gtid, int64_t gthreads) {
    if (p.key_bits == 8) pipe_stream_kb<LP_OCT_U, 8>(p, sm, bmask, lv, sq, gq, qcnt, abandon, gtid, gthreads);
    else pipe_stream_kb<4, 16>(p, sm, bmask, lv, sq, gq, qcnt, abandon, gtid, gthreads);
}

struct PipeExit {
    int k;            // last pass run
    int32_t ds, de;   // its appends [ds, de) (the old loop resumes at pass k + 1)
    int done;         // 1: fixpoint (or cap) reached, model written
};

// Runs key-space LEAD passes from pass 0 until the fixpoint (returns done = 1 after the
// epilogue) or until the auto schedule asks for STREAM passes (returns the state the
// unpipelined loop resumes from).  All threads of the CTA call it; the shared key
// summary of v_0 is already built.
struct LiveShared {      // the CTA's run table and live list (shared memory)
    const int4 *runs;
    int32_t *beg;
    int32_t *pre;
    int32_t *total;
};

__device__ __noinline__ PipeExit lm_pipe(const LMParams &p, uint32_t *sm, uint32_t *bmask,
                                         const Segment *segs, int32_t *squeue, int32_t n0,
                                         long long clk0, unsigned long long ns0, LiveShared ls) {
    __shared__ int32_t qcnt[2];
    __shared__ int32_t abandon;
    __shared__ int32_t s_t, s_queued;
    __shared__ unsigned long long s_vq, s_loaded;
    __shared__ int32_t s_nl;
    __shared__ int32_t s_sdone;   // pass 0: streaming warps done
    cg::grid_group grid = cg::this_grid();
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + tid;
    const int64_t gthreads = (int64_t)gridDim.x * blockDim.x;
    const bool lead = blockIdx.x == 0 && tid == 0;
    const int vbase = kStreamWarps * 32;
    const int nvt = (int)blockDim.x - vbase;             // verifier threads
    const bool verifier = tid >= vbase;
    const int vtid = tid - vbase;
    int32_t *gq[2] = {p.qbuf + (int64_t)blockIdx.x * p.qcap,
                      p.qbuf + ((int64_t)gridDim.x + blockIdx.x) * p.qcap};
    int32_t *sq[2] = {squeue, squeue + kPipeSq};
#define PDBG(k, i) p.dbg[((k) * gridDim.x + blockIdx.x) * 8 + (i)]
    if (tid == 0) {
        qcnt[0] = qcnt[1] = 0;
        abandon = 0;
        s_loaded = 0;
        s_nl = 0;
        s_sdone = 0;
    }
    for (int32_t i = tid; i < kPipeSq; i += blockDim.x) sq[0][i] = -1;   // (pass 0: not yet written)
    __syncthreads();
    // ---- pass 0: S_0 streamed by the streaming warps and verified by the verifier warps
    // as it appears in the shared queue (-1 = reserved, not yet written); the global part
    // of the queue is verified by all threads after the stream
    if (p.dbg && tid == 0) PDBG(0, 0) = PDBG(0, 1) = globaltimer();
    if (lead) {
        p.cand[1] = 0;
        p.vent[1] = 0;
        p.pcnt[1] = 0;
    }
    {
        const PassCtx c{p.buf0, p.buf1, sm, nullptr, nullptr, 0, bmask, segs, nullptr, p.pcnt, n0};
        int loaded = 0;
        if (!verifier) {
            const LiveList lv{ls.beg, ls.pre, *ls.total};   // (built before the call)
            if (blockIdx.x == 0 && tid == 0 && p.stats)
                atomicAdd(p.stats + 0, (unsigned long long)lv.total * (p.key_bits == 8 ? 10ull : 17ull));
            pipe_stream(p, sm, bmask, lv, sq[0], gq[0], &qcnt[0], &abandon, (int64_t)blockIdx.x * vbase + tid,
                        (int64_t)gridDim.x * vbase);
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();
                atomicAdd(&s_sdone, 1);
            }
        } else {
            for (int32_t i = vtid; i < kPipeSq; i += nvt) {
                bool have = false;
                for (;;) {   // wait until entry i is reserved, or the stream is over
                    if (i < *(volatile int32_t *)&qcnt[0]) { have = true; break; }
                    if (*(volatile int32_t *)&s_sdone == kStreamWarps) {
                        __threadfence_block();
                        have = i < *(volatile int32_t *)&qcnt[0];
                        break;
                    }
                    __nanosleep(64);
                }
                if (!have) break;
                int32_t s;
                while ((s = *(volatile int32_t *)&sq[0][i]) < 0) __nanosleep(32);
                loaded += verify_slot<false>(p, c, s, 0);
            }
        }
        __syncthreads();
        if (p.dbg && tid == 0) PDBG(0, 2) = globaltimer();
        const int32_t nc = min(qcnt[0], p.qcap + kPipeSq);
        for (int32_t i = kPipeSq + tid; i < nc; i += blockDim.x) loaded += verify_slot<false>(p, c, pipe_qget(sq[0], gq[0], i), 0);
        for (int o = 16; o; o >>= 1) loaded += __shfl_xor_sync(0xFFFFFFFFu, loaded, o);
        if (lane == 0 && loaded) atomicAdd(&s_loaded, (unsigned long long)loaded);
        __syncthreads();
        if (tid == 0) {
            if (nc) atomicAdd(p.cand + 0, nc);
            if (s_loaded) {
                atomicAdd(p.vent + 0, s_loaded);
                if (p.stats) atomicAdd(p.stats + 3, s_loaded);
            }
            s_loaded = 0;
        }
        if (p.dbg && tid == 0) PDBG(0, 3) = PDBG(0, 4) = globaltimer();
    }
    grid.sync();
    if (p.dbg && tid == 0) PDBG(0, 5) = globaltimer();
    const PassCounts pc0 = cta_pass_counts(p.pcnt + 0, p.cand + 0, p.vent + 0);
    int32_t t = n0 + pc0.appended;
    int32_t queued = pc0.queued;
    unsigned long long vq = pc0.vent;
    int32_t ds = n0, de = n0;
    for (int k = 0;; ++k) {
        // ---- pass k is complete: [de, t) are its appends
        const uint32_t *wr_k = (k & 1) ? p.buf0 : p.buf1;
        if (lead && p.stats) {
            atomicAdd(p.stats + 0, 4ull * (unsigned long long)queued + 12ull * (unsigned long long)(t - de));
            atomicAdd(p.stats + 1, 1ull);   // (reductions: no load on the lead thread's
            atomicAdd(p.stats + 2, (unsigned long long)queued);   //  critical path)
        }
        if (t == de || k + 1 >= p.max_passes || k + 1 == p.user_cap) {
            if (lead) {
                *p.iters_out = k + 1;
                if (t != de) atomicOr(p.status_out, k + 1 == p.user_cap ? kStCapped : kStGuard);
                if (p.status_user) *p.status_user = atomicOr(p.status_out, 0);
                if (p.stats) {
                    atomicAdd(p.stats + 0, 4ull * p.stats[3]);
                    p.stats[4] = (unsigned long long)(clock64() - clk0);
                    p.stats[5] = globaltimer() - ns0;
                }
            }
            if (p.dbg && tid == 0) p.dbg[(gridDim.x + blockIdx.x) * 8 + 6] = globaltimer();
            lm_extract(p, gtid, gthreads, wr_k);
            if (p.dbg) {
                __syncthreads();
                if (tid == 0) p.dbg[(gridDim.x + blockIdx.x) * 8 + 7] = globaltimer();
            }
            return PipeExit{k, de, t, 1};
        }
        if (lead && p.pops && k + 1 < p.pop_cap) p.pops[k + 1] = t;
        if (p.pass_mode == 0 &&
            ((int64_t)queued * p.dense_div > p.n_slots || (long long)vq * 8 > p.stream_entries))
            return PipeExit{k, de, t, 0};   // the auto schedule switches to STREAM passes
        // ---- Δ_k into the key summary: summary(v_{k+1})
        if (k == 0) add_to_shared<false>(p, sm, bmask, de, t, true);   // (later: in the phase)
        if (tid == 0) {
            qcnt[(k + 1) & 1] = 0;   // (S_{k+1} half: verified in phase k, streamed into next)
            abandon = 0;
        }
        __syncthreads();
        // the live runs of summary(v_{k+1}) (the verifier warps fold Δ_{k+1} into the summary
        // only after this phase's barrier, and the rows of its new lead atoms come from the
        // lead-occurrence lists, so the list need not follow them)
        build_live(p, bmask, ls.runs, ls.beg, ls.pre, ls.total);
        __syncthreads();
        const LiveList lv{ls.beg, ls.pre, *ls.total};
        if (lead && p.stats)   // (this phase's stream: pass k+2's candidates)
            atomicAdd(p.stats + 0, (unsigned long long)lv.total * (p.key_bits == 8 ? 10ull : 17ull));
        ds = de;
        de = t;
        // ---- phase j = k + 1
        const int j = k + 1;
        if (p.dbg && tid == 0 && j < 16) PDBG(j, 0) = globaltimer();
        const uint32_t *rd = (j & 1) ? p.buf1 : p.buf0;
        uint32_t *wr = (j & 1) ? p.buf0 : p.buf1;
        if (blockIdx.x == 0 && tid == 0) {
            p.cand[(j + 1) % 3] = 0;
            p.vent[(j + 1) % 3] = 0;
            p.pcnt[(j + 1) % 3] = 0;
        }
        const PassCtx c{rd, wr, sm, nullptr, nullptr, j, bmask, segs, nullptr, p.pcnt + j % 3, de};
        const int h = (j + 1) & 1;
        const int32_t nc = min(qcnt[h], p.qcap + kPipeSq);
        // pass j's verification by nt of the CTA's threads (ti = index among them)
        auto verify_pass = [&](int ti, int nt) {
            // wr still holds v_{j-1}: add Δ_{j-1} (spread over all CTAs)
            for (int64_t i = ds + (int64_t)ti * gridDim.x + blockIdx.x; i < de; i += (int64_t)gridDim.x * nt) {
                const int32_t a = __ldcg(p.order + i);
                atomicOr(wr + (a >> 5), 1u << (a & 31));
            }
            int loaded = 0, nl = 0;
            for (int32_t i = ti; i < nc; i += nt) loaded += verify_slot<false>(p, c, pipe_qget(sq[h], gq[h], i), 0);
            // rows whose lead atom became true in pass j - 1 (a warp per atom)
            const int nw = nt >> 5;
            for (int64_t i = ds + (int64_t)blockIdx.x * nw + (ti >> 5); i < de; i += (int64_t)gridDim.x * nw) {
                const int32_t a = __ldcg(p.order + i);
                const int32_t o0 = __ldg(p.locc_ptr + a), o1 = __ldg(p.locc_ptr + a + 1);
                for (int32_t o = o0 + lane; o < o1; o += 32) {
                    loaded += verify_slot<false>(p, c, __ldg(p.locc_slot + o), 0);
                    ++nl;
                }
            }
            for (int o = 16; o; o >>= 1) {
                loaded += __shfl_xor_sync(0xFFFFFFFFu, loaded, o);
                nl += __shfl_xor_sync(0xFFFFFFFFu, nl, o);
            }
            if (lane == 0) {
                if (loaded) atomicAdd(&s_loaded, (unsigned long long)loaded);
                if (nl) atomicAdd(&s_nl, nl);
            }
        };
        // pass 1 verifies S_1 = S_0 (pass 0's whole candidate set again) with every thread
        // before its stream starts; later passes' sets are verified by the verifier warps
        // beside the stream
        if (j == 1) {
            verify_pass(tid, blockDim.x);
            __syncthreads();
        }
        if (verifier) {
            if (j != 1) verify_pass(vtid, nvt);
            asm volatile("bar.sync 1, %0;" ::"r"(nvt) : "memory");   // the verifier warps
            if (vtid == 0) {
                if (nc + s_nl) atomicAdd(p.cand + j % 3, nc + s_nl);
                if (s_loaded) {
                    atomicAdd(p.vent + j % 3, s_loaded);
                    if (p.stats) atomicAdd(p.stats + 3, s_loaded);
                }
                if (p.dbg && j < 16) PDBG(j, 3) = PDBG(j, 4) = globaltimer();
                if (p.dbg && j >= 3 && j < 16) {   // (slots 6, 7: this CTA's S_j and locc rows)
                    PDBG(j, 6) = (unsigned long long)nc;
                    PDBG(j, 7) = (unsigned long long)s_nl;
                }
                s_loaded = 0;
                s_nl = 0;
                __threadfence();
                atomicAdd(p.pbar, 1u);                                   // arrive (pass j)
                const uint32_t target = (uint32_t)j * gridDim.x;
                while (ld_acquire_u32(p.pbar) < target) {}
                if (p.dbg && j < 16) PDBG(j, 5) = globaltimer();
                const int32_t tj = de + __ldcg(p.pcnt + j % 3);
                const int32_t qj = __ldcg(p.cand + j % 3);
                const unsigned long long vj = __ldcg(p.vent + j % 3);
                s_t = tj;
                s_queued = qj;
                s_vq = vj;
                if (tj == de || j + 1 >= p.max_passes || j + 1 == p.user_cap ||
                    (p.pass_mode == 0 && ((int64_t)qj * p.dense_div > p.n_slots || (long long)vj * 8 > p.stream_entries)))
                    abandon = 1;   // the stream running now will not be used
            }
            // Δ_j into the key summary right away, while S_{j+1} is still being streamed
            // against it: a row the stream then queues for a lead atom of Δ_j is also
            // reached through locc(Δ_j) -- verified twice, same result -- and the summary
            // stays a superset of summary(v_j), so S_{j+1} misses nothing
            asm volatile("bar.sync 1, %0;" ::"r"(nvt) : "memory");
            if (!*(volatile int32_t *)&abandon) {
                const int32_t tj = *(volatile int32_t *)&s_t;
                for (int32_t i0 = de + vtid; i0 < tj; i0 += 4 * nvt) {
                    uint32_t a[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int32_t i = i0 + u * nvt;
                        a[u] = i < tj ? (uint32_t)__ldcg(p.korder + i) : 0xFFFFFFFFu;
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (a[u] != 0xFFFFFFFFu) {
                            const uint32_t g = a[u] >> p.kshift;
                            atomicOr(sm + (g >> 5), 1u << (g & 31));
                            const uint32_t bk = g >> p.key_bits;
                            set_bucket(bmask, bk);
                        }
                }
            }
        } else {
            // pass j+1's candidates: rows whose lead key is in summary(v_j)
            const int64_t sgtid = (int64_t)blockIdx.x * vbase + tid;
            pipe_stream(p, sm, bmask, lv, sq[j & 1], gq[j & 1], &qcnt[j & 1], &abandon, sgtid,
                        (int64_t)gridDim.x * vbase);
            if (p.dbg && j < 16 && lane == 0) atomicMax(&PDBG(j, 2), globaltimer());
        }
        __syncthreads();
        if (p.dbg && tid == 0 && j < 16) PDBG(j, 1) = globaltimer();   // (phase over)
        t = s_t;
        queued = s_queued;
        vq = s_vq;
        k = j - 1;   // (the loop's ++k makes it j)
    }
#undef PDBG
}

// Estimated rows a key-mode LEAD pass would queue: Σ over live runs of rows x (set
// summary bits of the run's bucket / groups per bucket).  All threads of the CTA call it
// (the key summary in sm, 16-bit codes: bucket b = summary words [b << 11, (b+1) << 11)).
__device__ __noinline__ bool lead_start_too_dense(const LMParams &p, const uint32_t *sm, const int4 *runs_sm) {
    __shared__ uint32_t bc[32];
    __shared__ unsigned long long est;
    const int tid = threadIdx.x, lane = tid & 31;
    if (tid < 32) bc[tid] = 0u;
    if (tid == 0) est = 0ull;
    __syncthreads();
    // each warp counts a contiguous range of summary words (registers), flushing its sum
    // once per bucket (2048 words) it crosses: a few shared atomics per warp, not per word
    const int nwarps = blockDim.x >> 5, warp = tid >> 5;
    const int32_t per = ((p.ksm_words + nwarps - 1) / nwarps + 31) & ~31;   // (32-aligned: no chunk
                                                                          //  straddles a bucket)
    const int32_t w_lo = warp * per, w_hi = min(p.ksm_words, w_lo + per);
    uint32_t c = 0;
    int32_t cur_b = w_lo >> 11;
    for (int32_t w0 = w_lo; w0 < w_hi; w0 += 32) {
        const int32_t w = w0 + lane;
        if ((w0 >> 11) != cur_b) {   // (warp-uniform: w0 is)
            for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
            if (lane == 0 && c) atomicAdd(&bc[cur_b & 31], c);
            c = 0;
            cur_b = w0 >> 11;
        }
        c += w < w_hi ? (uint32_t)__popc(sm[w]) : 0u;
    }
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
    if (lane == 0 && c) atomicAdd(&bc[cur_b & 31], c);
    __syncthreads();
    for (int32_t r = tid; r < p.nruns; r += blockDim.x) {
        const int4 ru = runs_sm[r];
        const unsigned long long e = (unsigned long long)ru.y * 8ull * bc[ru.z & 31] >> 16;
        if (e) atomicAdd(&est, e);
    }
    __syncthreads();
    return (long long)est * p.dense_div > p.n_slots;
}

// One cooperative launch = the whole fixpoint loop of Algorithm 1:
// pass k reads v_k (rd) and writes v_{k+1} (wr); the loop ends after the first pass
// that derives nothing (u = v), and iters = k + 1 counts that pass too.
//
// Each pass is either a LEAD pass (lead atoms streamed, survivors queued and verified)
// or a STREAM pass (every body position streamed; the test is complete in EXACT mode,
// summary survivors are queued).  Both compute exactly θ(M v_k); the schedule only
// decides which bytes are read (p.pass_mode).
// ARMED: the instantiation for calls whose LEAD passes are armed (LMParams.arec set, no key
// plane): the key-space LEAD machinery (key summary, live runs, pipelined / overlapped
// passes) compiles out, and with it its register pressure; the other instantiation keeps it
// and drops the armed code.  Both run STREAM passes and plane-streaming LEAD passes.
template <bool EXACT, bool ARMED>
__global__ void __launch_bounds__(kFullThreads, 1) lm_full_kernel(const __grid_constant__ LMParams p) {
    extern __shared__ __align__(16) uint32_t sm[];
    __shared__ int32_t qcount;
    __shared__ unsigned long long loaded_cta;
    __shared__ __align__(16) uint32_t bmask[kBucketWords];   // key mode: bucket b has a set summary bit
    __shared__ Segment ssegs[kMaxSmemSegs];
    __shared__ int32_t squeue[kSmemQueue];
    __shared__ int32_t streamers_done;
    __shared__ __align__(8) uint64_t fill_bar;
    __shared__ int4 runs_sm[kMaxRuns];              // key mode: the run table (LMParams.runs)
    __shared__ int32_t live_beg[kMaxRuns];          //   and this pass's live list
    __shared__ int32_t live_pre[kMaxRuns + 1];
    __shared__ int32_t live_tot;
    __shared__ int32_t a_n[2];                      // armed LEAD passes: entries of the two lists
    __shared__ int32_t a_over;                      //   and the pass's overflow flag
    // (armed kernel) the pass barrier: this CTA's appends and overflow, what the barrier
    // word returned (the pass's appends, overflowing CTAs) and the previous pass's
    // schedule counts (loaded during this pass, one pass behind)
    __shared__ int32_t s_app, s_overflowed, s_bar_app, s_bar_over, s_q;
    __shared__ unsigned long long s_v;
    cg::grid_group grid = cg::this_grid();
    const int tid = threadIdx.x;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + tid;
    const int64_t gthreads = (int64_t)gridDim.x * blockDim.x;
    const bool lead = blockIdx.x == 0 && tid == 0;
    const LiveShared ls{runs_sm, live_beg, live_pre, &live_tot};
    if (p.dbg && tid == 0) p.dbg[blockIdx.x * 8 + 6] = globaltimer();
    __shared__ long long clk0;          // SM clock over the launch (lp_run.stats_out[4..5]);
    __shared__ unsigned long long ns0;  // in shared memory: no registers held across passes
    if (lead) {
        clk0 = clock64();
        ns0 = globaltimer();
    }

    bool lead_pass = starts_lead(p);
    bool keys = !ARMED && !EXACT && p.lead_codes && lead_pass;   // shared copy is in key space
    // v_0 = facts: the key summary and bucket mask images built at load are bulk-copied in
    // while the prologue runs (waited for after its barrier)
    const bool ksum_image = keys && !p.v0 && p.init_ksum;
    if (ksum_image && tid == 0) {
        mbar_init(&fill_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const uint32_t bytes = (uint32_t)p.ksm_words * 4u, bb = kBucketWords * 4u;
        mbar_expect_tx(&fill_bar, bytes + bb);
        constexpr uint32_t kChunk = 32768;
        for (uint32_t o = 0; o < bytes; o += kChunk)
            bulk_g2s_plain(reinterpret_cast<char *>(sm) + o, reinterpret_cast<const char *>(p.init_ksum) + o,
                           bytes - o < kChunk ? bytes - o : kChunk, &fill_bar);
        bulk_g2s_plain(bmask, p.init_ksum + p.ksm_words, bb, &fill_bar);
    }
    // (armed LEAD passes in summary mode keep no copy of v_k in shared memory: no summary)
    lm_prologue(p, !EXACT && !(ARMED && p.arec && starts_lead(p)), gtid, gthreads);   // v_0 (row a3), in-kernel
    if (gtid == 0) {
        p.cand[0] = 0;
        p.cand[1] = 0;
        p.cand[2] = 0;
        p.vent[0] = p.vent[1] = p.vent[2] = 0;
        if (p.stats)
            for (int i = 0; i < 6; ++i) p.stats[i] = 0;
    }
    grid.sync();
    if (p.dbg && tid == 0) p.dbg[(2 * gridDim.x + blockIdx.x) * 8 + 6] = globaltimer();
    const int32_t n0 = cta_pass_counts(p.tail, nullptr, nullptr).appended;
    __shared__ int32_t s_n0;   // (read again in the pass loop: not held in a register)
    if (tid == 0) s_n0 = n0;
    {
        if (!ksum_image)
            for (int32_t w = tid; w < kBucketWords; w += blockDim.x) bmask[w] = 0u;
        if (p.nseg <= kMaxSmemSegs)
            for (int32_t s = tid; s < p.nseg; s += blockDim.x) ssegs[s] = p.segs[s];
        if (keys)
            for (int32_t r = tid; r < p.nruns; r += blockDim.x) runs_sm[r] = __ldg(p.runs + r);
        if (ksum_image) {
            mbar_wait(&fill_bar, 0);
        } else if (keys) {   // key summary of v_0 straight from the initial list (bucket b =
                             // summary words [b << 11, (b + 1) << 11))
            int4 *s4 = reinterpret_cast<int4 *>(sm);
            for (int32_t w = tid; w < (p.ksm_words >> 2); w += blockDim.x) s4[w] = make_int4(0, 0, 0, 0);
            __syncthreads();
            add_to_shared<EXACT>(p, sm, bmask, 0, n0, true);
        } else {
            if (EXACT || !(ARMED && p.arec && lead_pass)) smem_fill(sm, EXACT ? p.buf0 : p.summary, p.sm_words);
        }
    }
    if (lead && p.pops && p.pop_cap > 0) p.pops[0] = n0;
    if (tid == 0) {
        qcount = 0;
        loaded_cta = 0;
        a_n[0] = a_n[1] = 0;
        a_over = 0;
        s_app = s_overflowed = s_bar_app = s_bar_over = s_q = 0;
        s_v = 0ull;
    }
    // armed LEAD passes (exact mode): every CTA keeps the rows
    // it armed -- lead atom in v_k, head not in v_k -- in a shared-memory list after the
    // truth words (two lists: the one verified and the one the survivors move to)
    bool armed = ARMED && p.arec != nullptr && lead_pass;   // (summary mode: the host passes no key plane then)
    int acur = 0;
    int32_t *const alist = reinterpret_cast<int32_t *>(sm + (EXACT ? p.sm_words : 0));
    if (keys) {   // the live runs of summary(v_0)
        __syncthreads();
        build_live(p, bmask, runs_sm, live_beg, live_pre, &live_tot);
        if (tid == 0) s_bmask_changed = 0;
    }
    __syncthreads();
    if (p.dbg && tid == 0) p.dbg[blockIdx.x * 8 + 7] = globaltimer();

    int32_t ds = n0, de = n0;  // atoms that became true in the previous pass
    int32_t dprev = n0;        // (the ds before that: the Δ size the arming loads were sized by)
    int k_start = 0;
    bool rebuild = false;                                // key space -> atom-id summary
    // Predictive start (auto schedule, 16-bit key plane): the rows a first LEAD pass would
    // queue are estimated from the live runs and the density of set bits in their buckets;
    // more than n_slots / dense_div -> start with STREAM passes instead of verifying them
    // (a v0 with many atoms outside D2 lights the coarse buckets: DESIGN.md "Schedule")
    // (v0 = NULL: the facts light only D2 buckets, never a dense start -- no estimate)
    if (!EXACT && keys && p.v0 && p.pass_mode == 0 && p.key_bits == 16 && p.nruns > 0 && p.predict &&
        lead_start_too_dense(p, sm, runs_sm)) {
        lead_pass = false;
        keys = false;
        rebuild = true;
    }
    // the live stream of a key-mode LEAD pass is long enough to hide verification and the
    // barrier behind it (else all warps stream, then all verify: fewer round trips per
    // row on the critical path -- DESIGN.md "Live runs")
    const long long oct_bytes = p.key_bits == 8 ? 10 : 17;
    if (!EXACT && keys && p.locc_ptr && (long long)live_tot * oct_bytes >= p.overlap_min_bytes) {
        // pipelined key-space LEAD passes
        const PipeExit e = lm_pipe(p, sm, bmask, p.nseg <= kMaxSmemSegs ? ssegs : p.segs, squeue, n0,
                                   lead ? clk0 : 0, lead ? ns0 : 0, ls);
        if (e.done) return;
        // the auto schedule switched: STREAM passes from pass e.k + 1 on (the summary is
        // rebuilt in atom-id space from v_{e.k+1})
        k_start = e.k + 1;
        ds = e.ds;
        de = e.de;
        lead_pass = false;
        keys = false;
        rebuild = true;
    }
    constexpr int kSpec = 4;
    uint32_t spec[kSpec];      // the next delta's first list entries, loaded with its count
    // (armed LEAD passes) this thread's Δ entry to arm, i = de + block + G * tid, and its arm
    // range: loaded right after the barrier beside the count (entries past it are ignored)
    int32_t arm_a = -1, arm_lo = 0, arm_hi = 0;
    __shared__ unsigned long long s_bprev[2];           // (armed kernel, thread 0) barrier words
    if (tid == 0) s_bprev[0] = s_bprev[1] = 0ull;      //   (first read after several syncs)
    int32_t lag_q = 0;                                  // (thread 0) the pass counts one pass behind
    unsigned long long lag_v = 0ull;
    for (int k = k_start;; ++k) {
        const uint32_t *rd = (k & 1) ? p.buf1 : p.buf0;
        uint32_t *wr = (k & 1) ? p.buf0 : p.buf1;
#define DBG_STAMP(i) p.dbg[(k * gridDim.x + blockIdx.x) * 8 + (i)]
#define DBG_NOW() (p.dbg_clock ? (unsigned long long)clock64() : globaltimer())
        if (p.dbg && tid == 0 && k < 16) DBG_STAMP(0) = DBG_NOW();
        if (p.overlap && !EXACT) {   // empty shared queue for this pass (last reader: before the barrier)
            for (int32_t i = tid; i < kSmemQueue; i += blockDim.x) squeue[i] = -1;
            if (tid == 0) streamers_done = 0;
            if (k == 0) __syncthreads();   // (later passes sync after the delta below)
        }
        if (k > 0 || rebuild) {
            // shared copy: v_{k-1} -> v_k
            if (EXACT && (de - ds) > (p.sm_words >> 2)) {
                for (int32_t w = tid; w < p.sm_words; w += blockDim.x) sm[w] = __ldcg(rd + w);
            } else if (!EXACT && rebuild) {
                // first STREAM pass after LEAD passes in key space: the atom-id summary of
                // v_k from the complete truth vector rd (bit g = OR of atoms g<<shift ..)
                rebuild = false;
                for (int32_t w = tid; w < p.sm_words; w += blockDim.x) sm[w] = 0u;
                __syncthreads();
                for (int32_t t = tid; t < p.nwords; t += blockDim.x) {
                    const uint32_t v = __ldcg(rd + t);
                    if (!v) continue;
                    if (p.shift >= 5) {
                        const uint32_t g = (uint32_t)t >> (p.shift - 5);
                        atomicOr(sm + (g >> 5), 1u << (g & 31));
                    } else {
                        for (uint32_t b = v; b;) {
                            const uint32_t g = ((uint32_t)t * 32u + (uint32_t)(__ffs(b) - 1)) >> p.shift;
                            b &= b - 1;
                            atomicOr(sm + (g >> 5), 1u << (g & 31));
                        }
                    }
                }
            } else if (!EXACT && armed && lead_pass) {
                // (armed summary mode: no shared copy of v_k to bring up to date)
            } else if (EXACT || keys) {
                // the first kSpec x blockDim entries were loaded right after the barrier
#pragma unroll
                for (int u = 0; u < kSpec; ++u) {
                    const int32_t i = ds + tid + u * (int32_t)blockDim.x;
                    if (i < de) {
                        // (an entry past the speculative bound was not loaded: load it now)
                        const uint32_t e = spec[u] != 0xFFFFFFFFu ? spec[u] : (uint32_t)__ldcg((EXACT ? p.order : p.korder) + i);
                        const uint32_t g = EXACT ? e : (e >> p.kshift);
                        atomicOr(sm + (g >> 5), 1u << (g & 31));
                        if (!EXACT && keys) {
                            const uint32_t bk = g >> p.key_bits;
                            set_bucket(bmask, bk);
                        }
                    }
                }
                add_to_shared<EXACT>(p, sm, bmask, ds + kSpec * (int32_t)blockDim.x, de, keys);
            } else {
                add_to_shared<EXACT>(p, sm, bmask, ds, de, keys);
            }
            if (p.dbg && !armed && tid == 0 && k >= 3 && k < 16) DBG_STAMP(6) = globaltimer();
            __syncthreads();
            if (keys && lead_pass && s_bmask_changed) {   // the live runs of summary(v_k)
                build_live(p, bmask, runs_sm, live_beg, live_pre, &live_tot);
                __syncthreads();
                if (tid == 0) s_bmask_changed = 0;   // (read again only after the next fold)
            }
            if (p.dbg && !armed && tid == 0 && k >= 3 && k < 16) DBG_STAMP(7) = globaltimer();
        }
        const LiveList lv{live_beg, live_pre, live_tot};
        if (lead && p.stats && keys && lead_pass)   // the pass's streamed bytes: codes + tag per live octet
            atomicAdd(p.stats + 0, (unsigned long long)lv.total * (p.key_bits == 8 ? 10ull : 17ull));
        // rows queued in pass k are counted in cand[k % 3]; the slot of pass k+1 was last
        // read before the previous barrier and is first written after the next one
        if (lead) {
            p.cand[(k + 1) % 3] = 0;
            p.vent[(k + 1) % 3] = 0;
            p.pcnt[(k + 1) % 3] = 0;
        }
        const PassCtx c{rd, wr, sm, p.qbuf + (int64_t)blockIdx.x * p.qcap, &qcount, k, bmask,
                        p.nseg <= kMaxSmemSegs ? ssegs : p.segs, squeue, p.pcnt + k % 3, de,
                        ARMED ? &s_app : nullptr};
        if (p.dbg && tid == 0 && k < 16) DBG_STAMP(1) = DBG_NOW();
        const int j0 = (EXACT && lead_pass) ? 1 : 0;
        int loaded = 0;
        // Overlapped LEAD pass: kStreamWarps warps stream, the others verify the shared
        // queue entries while they appear (an entry is written right after its slot is
        // reserved; -1 = not yet), so only the tail of the verification is left after
        // the stream.  Entries past the shared part wait for the epilogue.
        // (key mode only: with the exact in-smem truth the stream is L2-fast and 4 fewer
        // streaming warps cost more than the overlap saves -- measured C2 +20 %, C3 +6 %)
        const bool overlap = p.overlap && !EXACT && keys && (long long)lv.total * oct_bytes >= p.overlap_min_bytes;
        if (overlap) {
            const int warp = tid >> 5;
            const int64_t sthreads = (int64_t)gridDim.x * (kStreamWarps * 32);
            if (warp < kStreamWarps) {
                const int64_t sgtid = (int64_t)blockIdx.x * (kStreamWarps * 32) + tid;
                octets_lead(p, c, lv, sgtid, sthreads);
                __syncwarp();
                if ((tid & 31) == 0) {
                    __threadfence_block();
                    atomicAdd(&streamers_done, 1);
                }
            } else {
                const int vthreads = blockDim.x - kStreamWarps * 32;
                for (int32_t i = tid - kStreamWarps * 32; i < kSmemQueue; i += vthreads) {
                    bool have = false;
                    for (;;) {   // wait until entry i is reserved, or the stream is over
                        if (i < *(volatile int32_t *)&qcount) { have = true; break; }
                        if (*(volatile int32_t *)&streamers_done == kStreamWarps) {
                            __threadfence_block();
                            have = i < *(volatile int32_t *)&qcount;
                            break;
                        }
                        __nanosleep(64);
                    }
                    if (!have) break;
                    int32_t s;
                    while ((s = *(volatile int32_t *)&squeue[i]) < 0) __nanosleep(32);
                    loaded += verify_slot<EXACT>(p, c, s, j0);
                }
            }
        }
        else if (!EXACT && keys) octets_lead(p, c, lv, gtid, gthreads);
        else if (lead_pass && armed) {
            // arm the rows led by the atoms that became true in the previous pass (pass 0: the
            // atoms of v_0); Δ entry i is armed by CTA (i - a0) mod G.  A full list verifies a
            // row at once and marks the pass: its survivors cannot be kept, so the next LEAD
            // passes stream the planes instead (the count of rows queued carries the mark)
            int32_t *const L0 = alist + (int64_t)acur * p.arm_cap;
            int32_t *const L1 = alist + (int64_t)(acur ^ 1) * p.arm_cap;
            auto arm = [&](int32_t lo, int32_t hi) {
                if (hi <= lo) return;
                // (the records are verified after the block barrier below, by other threads:
                // start their cold lines toward L2 now, 4 records per line, up to 8 lines)
                if (p.prefetch)
                    for (int32_t o = lo & ~3, n = 0; o < hi && n < 8; o += 4, ++n) prefetch_l2(p.arec + 2 * (int64_t)o);
                int32_t pos = atomicAdd(&a_n[acur], hi - lo);
                for (int32_t o = lo; o < hi; ++o, ++pos) {
                    if (pos < p.arm_cap) {
                        L0[pos] = o;
                    } else {
                        a_over = 1;
                        armed_verify<EXACT>(p, c, o, loaded);
                    }
                }
            };
            // (measured: arming from the list entries already loaded for the fold, instead of
            // loading them again here, was slower -- C3 7.81 vs 7.60 ms)
            // Δ entry i is armed by thread (i - a0) / G of CTA (i - a0) mod G, which also ORs the
            // atom into wr (the buffer that still holds v_{k-1}: see below)
            {
                const int32_t a0 = k == 0 ? 0 : ds, a1 = k == 0 ? s_n0 : de;
                int64_t i = a0 + blockIdx.x + (int64_t)gridDim.x * tid;
                if (k > 0 && tid <= 2 * ((ds - dprev) / (int32_t)gridDim.x) + 1) {   // the first entry
                    if (i < a1) {                                                     // came with the barrier
                        if (EXACT) {   // (its range, looked up now: see the barrier)
                            arm_lo = __ldg(p.arm_ptr + arm_a);
                            arm_hi = __ldg(p.arm_ptr + arm_a + 1);
                        }
                        arm(arm_lo, arm_hi);
                        atomicOr(wr + (arm_a >> 5), 1u << (arm_a & 31));
                    }
                    i += gthreads;
                }
                for (; i < a1; i += gthreads) {
                    const int32_t a = __ldcg(p.order + i);
                    arm(__ldg(p.arm_ptr + a), __ldg(p.arm_ptr + a + 1));
                    if (k > 0) atomicOr(wr + (a >> 5), 1u << (a & 31));
                }
            }
            if (p.dbg && k < 16 && (tid & 31) == 0) atomicMax(&DBG_STAMP(6), DBG_NOW());   // arming done
            __syncthreads();
            if (p.dbg && tid == 0 && k < 16) DBG_STAMP(7) = DBG_NOW();   // verification starts
            const int32_t na = min(a_n[acur], p.arm_cap);
            for (int32_t i = tid; i < na; i += blockDim.x) {
                const int32_t o = L0[i];
                if (armed_verify<EXACT>(p, c, o, loaded)) L1[atomicAdd(&a_n[acur ^ 1], 1)] = o;   // (< na)
            }
            __syncthreads();
            if (tid == 0) {   // (the overflow mark: carried by the pass barrier)
                if (na) atomicAdd(p.cand + k % 3, na);
                if (a_over) s_overflowed = 1;
                if (p.stats && na) {   // (this CTA's share: the counts reach the lead a pass late)
                    atomicAdd(p.stats + 0, 36ull * (unsigned long long)na);   // record + its list entry
                    atomicAdd(p.stats + 2, (unsigned long long)na);
                }
                a_n[acur] = 0;
                a_over = 0;
            }
            acur ^= 1;
        }
        else if (EXACT && lead_pass && p.xlead16) octets_exact16<4>(p, c, gtid, gthreads);
        else if (EXACT && lead_pass && p.lead32) flat_lead_exact<4>(p, c, gtid, gthreads);
        else if (lead_pass) all_segments<EXACT, true>(p, c, gtid, gthreads);
        else {
            int sl = all_segments<EXACT, false>(p, c, gtid, gthreads);   // int4 loads issued
            if (p.stats) {
                for (int o = 16; o; o >>= 1) sl += __shfl_xor_sync(0xFFFFFFFFu, sl, o);
                if ((tid & 31) == 0 && sl) atomicAdd(p.stats + 0, 16ull * (unsigned long long)sl);
            }
        }
        if (p.dbg && k < 16 && (tid & 31) == 0) atomicMax(&DBG_STAMP(2), DBG_NOW());
        // wr still holds v_{k-1}: add the atoms derived in pass k-1 so that it is a superset
        // of v_k before the barrier (nobody reads wr during pass k -- emit_head tests the
        // head against v_k first -- so this is off the critical path at the pass top);
        // spread over all CTAs
        if (!(lead_pass && armed))   // (an armed pass did it while arming)
            for (int64_t i = ds + (int64_t)tid * gridDim.x + blockIdx.x; i < de; i += gthreads) {
                const int32_t a = __ldcg(p.order + i);
                atomicOr(wr + (a >> 5), 1u << (a & 31));
            }
        if (lead_pass && armed) {   // (an armed pass queues nothing: only its verified entries)
            for (int o = 16; o; o >>= 1) loaded += __shfl_xor_sync(0xFFFFFFFFu, loaded, o);
            if ((tid & 31) == 0 && loaded) atomicAdd(&loaded_cta, (unsigned long long)loaded);
        } else if (!EXACT || lead_pass) {  // epilogue: verify this CTA's queued rows
            __syncthreads();
            const int32_t nc = min(qcount, p.qcap + kSmemQueue);
            __syncthreads();
            if (tid == 0) {
                qcount = 0;
                if (nc) atomicAdd(p.cand + k % 3, nc);
            }
            for (int32_t i = (overlap ? min(nc, kSmemQueue) : 0) + tid; i < nc; i += blockDim.x)
                loaded += verify_slot<EXACT>(p, c, qget(c, i), j0);
            for (int o = 16; o; o >>= 1) loaded += __shfl_xor_sync(0xFFFFFFFFu, loaded, o);
            if ((tid & 31) == 0 && loaded) atomicAdd(&loaded_cta, (unsigned long long)loaded);
        }
        if (p.dbg && k < 16) {
            if ((tid & 31) == 0) atomicMax(&DBG_STAMP(3), DBG_NOW());
            __syncthreads();
            if (tid == 0) DBG_STAMP(4) = DBG_NOW();
        }
        __syncthreads();
        if (tid == 0 && loaded_cta) {   // body entries the verification loaded (schedule + stats)
            atomicAdd(p.vent + k % 3, loaded_cta);
            if (p.stats) atomicAdd(p.stats + 3, loaded_cta);
            loaded_cta = 0;
        }
        // split model output: the prologue's PCIe stores of v_0's words are ordered before
        // the epilogue's stores of the same words by one system fence per CTA (cumulative
        // over the CTA's stores after the block barrier above) at the end of pass 2 --
        // by then they have long completed, so it costs nothing; shorter runs fence below
        if (p.model_split && k == kSplitFencePass && tid == 0) __threadfence_system();
        if constexpr (ARMED) {
            // The pass barrier of the armed kernel: one 64-bit reduction per CTA on the word
            // of this pass's parity, [arrivals:24 | overflowing CTAs:8 | appends:32] (both
            // fields only grow within a call, per word: differences to the word's last value
            // are this pass's), released after the block barrier above (cumulative over the
            // CTA's writes) and polled with acquire -- the pass's append count arrives with
            // the barrier instead of being read back from the hot counter line after it.
            if (tid == 0) {
                unsigned long long add = (1ull << 40) | (unsigned long long)(uint32_t)s_app;
                if (s_overflowed) add += 1ull << 32;
                asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p.lbar + (k & 1)), "l"(add) : "memory");
                const uint32_t target = (uint32_t)((((unsigned long long)(k / 2) + 1ull) * gridDim.x) & 0xFFFFFFull);
                unsigned long long v;
                for (;;) {
                    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p.lbar + (k & 1)) : "memory");
                    if ((((uint32_t)(v >> 40) - target) & 0xFFFFFFu) < 0x800000u) break;
                }
                const unsigned long long pv = s_bprev[k & 1];
                s_bar_app = (int32_t)((uint32_t)v - (uint32_t)pv);
                s_bar_over = (int32_t)((((v >> 32) & 0xFFull) - ((pv >> 32) & 0xFFull)) & 0xFFull);
                s_bprev[k & 1] = v;
                s_app = 0;
                s_overflowed = 0;
                s_q = lag_q;    // the previous pass's counts, loaded during this one
                s_v = lag_v;
            }
            __syncthreads();
        } else {
            grid.sync();
        }
        if (p.dbg && tid == 0 && k < 16) DBG_STAMP(5) = DBG_NOW();
#undef DBG_STAMP
#undef DBG_NOW
        // after the barrier: this pass's appends (a slot nobody touches again before the
        // next barrier -- the shared tail would race with the next pass's appends)
        if (EXACT || keys) {
            // load the first list slots of this pass's appends together with their count
            // instead of after it (one L2 round trip less before the next stream); slots at
            // or past the count are not used (the next pass may be appending there already)
            const int32_t *lst = EXACT ? p.order : p.korder;
            // (speculative: only up to about twice the last delta -- every CTA loads the same
            // entries, so loads past the count queue on the same L2 lines for nothing;
            // 0xFFFFFFFF = not loaded)
            const int32_t spec_n = 2 * (de - ds) + 256;
#pragma unroll
            for (int u = 0; u < kSpec; ++u) {
                const int32_t d = tid + u * (int32_t)blockDim.x;
                const int32_t i = de + d;
                spec[u] = (d < spec_n && i < p.n_order_cap) ? (uint32_t)__ldcg(lst + i) : 0xFFFFFFFFu;
            }
        }
        if (armed && lead_pass) {
            // (only as many threads as twice the last Δ needs: the loads past the count are
            // wasted L2 requests)
            const int64_t i = de + blockIdx.x + (int64_t)gridDim.x * tid;
            const bool want = tid <= 2 * ((de - ds) / (int32_t)gridDim.x) + 1;
            arm_a = (want && i < p.n_order_cap) ? __ldcg(p.order + i) : -1;
        }
        // (the pass's counts are requested before anything waits on the entry above: both
        // round trips overlap)
        PassCounts pcs;
        if constexpr (ARMED) {   // (the appends came with the barrier; the schedule counts lag)
            pcs.appended = s_bar_app;
            pcs.queued = s_q;
            pcs.vent = s_v;
            if (tid == 0) {
                lag_q = __ldcg(p.cand + k % 3);
                lag_v = __ldcg(p.vent + k % 3);
            }
        } else {
            pcs = cta_pass_counts(p.pcnt + k % 3, p.cand + k % 3, p.vent + k % 3);
        }
        // summary mode: the arm range is looked up right away (no Δ fold follows to hide it:
        // measured C4 0.0665 vs 0.0707 ms); exact mode looks it up at arming time (a thread
        // waiting on its entry here would hold up the CTA's Δ fold: C3 8.08 vs 7.89 ms)
        if (!EXACT && armed && lead_pass) {
            if (arm_a >= 0 && arm_a < p.n_ext_atoms) {
                arm_lo = __ldg(p.arm_ptr + arm_a);
                arm_hi = __ldg(p.arm_ptr + arm_a + 1);
            }
        }

        const int32_t t = de + pcs.appended;
        const int32_t queued = pcs.queued;
        if (lead && p.stats) {
            // algorithmic bytes of this pass: the planes it streamed, 4 B per body entry
            // and head the verification loaded, the delta list read twice and the truth
            // words it ORs
            // (STREAM passes added the int4 loads they issued themselves, atomically)
            // (armed kernel: the verified rows were added by each CTA itself, see above)
            const unsigned long long qd = ARMED ? 0ull : (unsigned long long)queued;
            atomicAdd(p.stats + 0, (unsigned long long)(lead_pass && !keys ? (armed ? 12ull * (unsigned long long)(k == 0 ? s_n0 : de - ds) : p.lead_bytes) : 0) +
                                       4ull * qd + 12ull * (unsigned long long)(t - de));
            if (lead_pass) atomicAdd(p.stats + 1, 1ull);   // (reductions: no load on the
            atomicAdd(p.stats + 2, qd);                     //  lead thread's critical path)
        }
        if (t == de || k + 1 >= p.max_passes || k + 1 == p.user_cap) {  // u = v: fixpoint (or a cap)
            if (lead) {
                *p.iters_out = k + 1;
                if (t != de) atomicOr(p.status_out, k + 1 == p.user_cap ? kStCapped : kStGuard);
                if (p.status_user) *p.status_user = atomicOr(p.status_out, 0);
                if (p.stats) {
                    atomicAdd(p.stats + 0, 4ull * p.stats[3]);
                    p.stats[4] = (unsigned long long)(clock64() - clk0);
                    p.stats[5] = globaltimer() - ns0;
                }
            }
            if (p.dbg && tid == 0) p.dbg[(gridDim.x + blockIdx.x) * 8 + 6] = globaltimer();
            lm_zero_summaries(p, !EXACT, gtid, gthreads);
            if (p.model_split && k < kSplitFencePass) {   // (the fence above did not run yet)
                if (tid == 0) __threadfence_system();
                grid.sync();
            }
            lm_extract(p, gtid, gthreads, wr, s_n0, t);
            if (p.dbg) {
                __syncthreads();
                if (tid == 0) p.dbg[(gridDim.x + blockIdx.x) * 8 + 7] = globaltimer();
            }
            return;
        }
        if (lead && p.pops && k + 1 < p.pop_cap) p.pops[k + 1] = t;
        // auto schedule: STREAM from the first LEAD pass that queued more than 1/dense_div of
        // the rows or whose verification loaded more than 1/8 of the entries a STREAM pass
        // reads (a verified entry costs a 32-byte sector, a streamed one 4 bytes)
        const unsigned long long vq = pcs.vent;
        if (armed && s_bar_over > 0) {   // a list overflowed: stream from now on (summary
            armed = false;                   // mode: over the atom-id summary, built first)
            if (!EXACT) rebuild = true;
        }
        if (lead_pass && p.pass_mode == 0 &&
            ((int64_t)queued * p.dense_div > p.n_slots || (long long)vq * 8 > p.stream_entries)) {
            lead_pass = false;
            rebuild = keys || (!EXACT && armed) || rebuild;
            keys = false;
        }
        dprev = ds;
        ds = de;
        de = t;
    }
}

cudaError_t launch_lm_full(const LMParams &p, bool exact, int blocks, size_t smem, cudaStream_t st) {
    LMParams q = p;
    void *args[] = {(void *)&q};
    const bool armed = p.arec != nullptr;
    const void *k = exact ? (armed ? (const void *)lm_full_kernel<true, true> : (const void *)lm_full_kernel<true, false>)
                          : (armed ? (const void *)lm_full_kernel<false, true> : (const void *)lm_full_kernel<false, false>);
    return cudaLaunchCooperativeKernel(k, dim3(blocks), dim3(kFullThreads), args, smem, st);
}

// ------------------------------------------------------------------------------------
// least model: frontier (semi-naive) variant
// ------------------------------------------------------------------------------------

// Level-synchronous push: the atoms that became true at level k decrement the
// remaining-body counter of every row whose body contains them; a counter reaching 0
// means body(r) ⊆ I_k, so head(r) ∈ I_{k+1} -- the same stage as the full θ-pass, hence
// the same model, pass count and popcount trace (reading R6).
//
// The per-row counters hold the number of body atoms still unknown; the prologue sets
// them to the row's body length L segment by segment (coalesced, overlapping the v_0
// build), so the hot loop needs no length lookup and nothing has to be cleaned up.
template <bool CL>
__global__ void __launch_bounds__(kThreads, 1) lm_frontier_kernel(const __grid_constant__ LMParams p) {
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + tid;
    const int64_t gthreads = (int64_t)gridDim.x * blockDim.x;
    const int64_t gwarp = gtid >> 5;
    const int64_t nwarps = gthreads >> 5;
    lm_prologue(p, false, gtid, gthreads);
    for (int32_t s = 0; s < p.nseg; ++s) {   // counters <- L (4 rows per word in byte mode)
        const Segment sg = p.segs[s];
        // (nibbles: 8 rows per word -- segments are 8-aligned then, see abi.cu; bytes: 4)
        const uint32_t v = p.cnt_bits == 4 ? (uint32_t)sg.L * 0x11111111u
                         : p.cnt_bits == 8 ? (uint32_t)sg.L * 0x01010101u : (uint32_t)sg.L;
        const int64_t w0 = p.cnt_bits == 4 ? sg.slot_off >> 3 : p.cnt_bits == 8 ? sg.slot_off >> 2 : sg.slot_off;
        const int64_t nw = p.cnt_bits == 4 ? sg.count_pad >> 3 : p.cnt_bits == 8 ? sg.count_pad >> 2 : sg.count_pad;
        for (int64_t w = gtid; w < nw; w += gthreads) p.cnt[w0 + w] = v;
    }
    pass_barrier<CL>();
    const int32_t n0 = cta_pass_counts(p.tail, nullptr, nullptr).appended;
    const bool lead = blockIdx.x == 0 && tid == 0;
    if (lead && p.pops && p.pop_cap > 0) p.pops[0] = n0;
    // occurrences as (slot, head(slot), occ range of that head): a firing row's head is
    // queued for the next level together with its own occurrence range
    const int4 *occ = reinterpret_cast<const int4 *>(p.occ_slot);
    int4 *const fq0 = reinterpret_cast<int4 *>(p.fq);   // queue of level l: fq0 + (l & 1) * n_order_cap
    // level kk: push one newly true atom's occurrences; heads that become true go to the
    // queue of level kk + 1 (slot count in pcnt[kk % 3])
    auto push = [&](int32_t o0, int32_t o1, int kk) {
        for (int32_t o = o0 + lane; o < o1; o += 32) {
            const int4 e = __ldg(occ + o);
            const int32_t slot = e.x;
            bool fired;
            if (p.cnt_bits == 4) {    // a nibble never underflows: <= L <= 15 decrements
                const uint32_t sh = (uint32_t)(slot & 7) << 2;
                fired = ((atomicSub(p.cnt + (slot >> 3), 1u << sh) >> sh) & 0xFu) == 1u;
            } else if (p.cnt_bits == 8) {   // a byte never underflows: <= L decrements
                const uint32_t sh = (uint32_t)(slot & 3) << 3;
                fired = ((atomicSub(p.cnt + (slot >> 2), 1u << sh) >> sh) & 0xFFu) == 1u;
            } else {
                fired = atomicSub(p.cnt + slot, 1u) == 1u;
            }
            if (fired) {                                // body(r) ⊆ I_kk
                const int32_t h = e.y;
                const uint32_t bit = 1u << (h & 31);
                const uint32_t old = atomicOr(p.buf0 + (h >> 5), bit);
                if (!(old & bit)) {
                    const int32_t pos = atomicAdd(p.pcnt + kk % 3, 1);
                    LP_CHECK(pos < p.n_order_cap && slot >= 0 && slot < p.n_slots);
                    fq0[(int64_t)((kk + 1) & 1) * p.n_order_cap + pos] = make_int4(h, e.z, e.w, 0);
                    if (p.stage && h < p.n_out) p.stage[h] = kk + 1;
                    // h's occurrences are read at the next level, after the barrier: start
                    // their (cold) lines toward L2 now (up to 8 lines = 64 occurrences)
                    if (p.prefetch)
                        for (int32_t o = e.z & ~7, n = 0; o < e.w && n < 8; o += 8, ++n) prefetch_l2(occ + o);
                }
            }
        }
    };
    // level 0: the atoms of v_0 (the prologue's derivation list)
    if (lead) p.pcnt[1] = 0;
    for (int64_t i = gwarp; i < n0; i += nwarps) {
        const int32_t a = __ldcg(p.order + i);
        push((int32_t)__ldg(p.occ_ptr + a), (int32_t)__ldg(p.occ_ptr + a + 1), 0);
    }
    __shared__ int32_t s_cnt;
    int32_t total = n0;
    for (int k = 0;; ++k) {
        pass_barrier<CL>();
        // level k is complete; level j = k + 1 starts at once from its queue (entries are
        // -1 past its end: no count needed to start), while one thread per CTA fetches
        // level k's append count (termination, popcount trace) -- if it is 0 the queue
        // is empty and level j does nothing
        const int j = k + 1;
        const bool capped = j >= p.max_passes || j == p.user_cap;
        int4 *q = fq0 + (int64_t)(j & 1) * p.n_order_cap;
        int4 e0 = make_int4(-1, 0, 0, 0);
        if (!capped && gwarp < p.n_order_cap) e0 = __ldcg(q + gwarp);
        if (tid == 0) s_cnt = __ldcg(p.pcnt + k % 3);
        if (lead) p.pcnt[(j + 1) % 3] = 0;   // (level j appends to pcnt[j % 3])
        if (!capped)
            for (int64_t i = gwarp;; i += nwarps) {
                const int4 e = i == gwarp ? e0 : (i < p.n_order_cap ? __ldcg(q + i) : make_int4(-1, 0, 0, 0));
                if (e.x < 0) break;
                if (lane == 0) q[i].x = -1;   // consumed (the queue is reused two levels on)
                push(e.y, e.z, j);
            }
        __syncthreads();
        const int32_t cnt = s_cnt;
        if (cnt == 0 || capped) {
            if (lead) {
                *p.iters_out = k + 1;
                if (cnt != 0) atomicOr(p.status_out, k + 1 == p.user_cap ? kStCapped : kStGuard);
                if (p.status_user) *p.status_user = atomicOr(p.status_out, 0);
            }
            if (capped)   // level j's queue was not consumed
                for (int64_t i = gtid; i < cnt; i += gthreads) q[i].x = -1;
            lm_extract(p, gtid, gthreads, p.buf0);
            return;
        }
        total += cnt;
        if (lead && p.pops && k + 1 < p.pop_cap) p.pops[k + 1] = total;
    }
}

// Launch a kernel either cooperatively over `blocks` CTAs or as ONE cluster of `cluster` CTAs.
template <class K>
static cudaError_t launch_grid_or_cluster(K kernel_grid, K kernel_cluster, const void *param, size_t psize,
                                          int blocks, int cluster, size_t smem, cudaStream_t st,
                                          int cl_threads = 0) {
    (void)psize;
    void *args[] = {const_cast<void *>(param)};
    if (cluster <= 0)
        return cudaLaunchCooperativeKernel((const void *)kernel_grid, dim3(blocks), dim3(kThreads), args, smem, st);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)cluster);
    cfg.blockDim = dim3((unsigned)(cl_threads > 0 ? cl_threads : kThreads));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)cluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelExC(&cfg, (const void *)kernel_cluster, args);
}

cudaError_t launch_lm_frontier(const LMParams &p, int blocks, cudaStream_t st, int cluster) {
    LMParams q = p;
    return launch_grid_or_cluster(lm_frontier_kernel<false>, lm_frontier_kernel<true>, &q, sizeof(q), blocks,
                                  cluster, 0, st, p.fr_cl_threads);
}

// ------------------------------------------------------------------------------------
// least model: ONE thread-block cluster for programs whose truth vector fits shared memory
// ------------------------------------------------------------------------------------
//
// Small exact-mode programs are latency-bound on the persistent grid (a 148-CTA grid
// barrier, counters in L2, dependent L2 round trips per pass: C1 ~7 us per pass).  Here a
// cluster of S CTAs runs the whole fixpoint: every CTA keeps v_k and v_{k+1} EXACTLY in
// its shared memory and streams its share of the flat lead / head planes (LEAD pass: a row
// whose lead atom is in v_k and whose head is not is queued in shared memory); the queue
// is verified after the stream by all threads (the other body atoms: one round trip,
// tested in shared memory) and a firing head is ORed into the CTA's own v_{k+1} (a
// shared-memory atomic).  Then every CTA ORs the words its pass changed into the other
// CTAs' v_{k+1} (distributed shared memory, fire-and-forget reductions), one cluster
// barrier (release / acquire) makes them visible, and every CTA -- holding the same
// complete v_{k+1} -- counts the new atoms (u != v, the popcount trace) on its own and
// writes the stages of the new atoms in the words it owns (word w: CTA w mod S).  The
// buffer that held v_k is brought up to v_{k+1} at the next pass top (atomicOr: the next
// pass's remote ORs may already arrive; ORs commute).  Same θ(M v_k) per pass as the
// other kernels: same model, iters, popcounts, stages.
constexpr int kClQueue = 4096;   // candidate rows a CTA queues per pass (shared memory)

// The other body atoms of a queued row (lead in v_k, head not): one round trip for up to 8
// of them, tested exactly against v_k; a firing row's head goes into this CTA's v_{k+1}.
__device__ __forceinline__ void cl_verify(const LMParams &p, const Segment *segs, const int32_t *colg,
                                          const int32_t *heads, const uint32_t *rd, uint32_t *wr, int32_t slot) {
    int lo = 0, hi = p.nseg - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (segs[mid].slot_off <= slot) lo = mid; else hi = mid - 1;
    }
    const int32_t L = segs[lo].L;
    const int64_t cp = segs[lo].count_pad;
    const int32_t *colp = colg + segs[lo].col_off + (slot - segs[lo].slot_off);
    const int32_t h = heads[slot];
    bool ok = true;
    for (int32_t j0 = 1; j0 < L && ok; j0 += 8) {
        uint32_t x[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = j0 + j < L ? (uint32_t)colp[(int64_t)(j0 + j) * cp] : 0xFFFFFFFFu;
#pragma unroll
        for (int j = 0; j < 8; ++j) ok = ok && (x[j] == 0xFFFFFFFFu || sm_bit(rd, x[j]));
    }
    if (ok) atomicOr(wr + (h >> 5), 1u << (h & 31));
}

// U = quads of the lead / head planes in flight per thread (1 when the cluster has at most
// two quads per thread: the unrolled padding would only add instructions)
template <int U>
__global__ void __launch_bounds__(kThreads, 1) lm_cluster_kernel(const __grid_constant__ LMParams p) {
    extern __shared__ __align__(16) uint32_t cbuf[];
    __shared__ int32_t s_cnt[2], s_qn[2];   // per pass parity: reset one pass ahead (fewer barriers)
    __shared__ int32_t cl_q[kClQueue];     // this pass's candidate rows
    __shared__ Segment ssegs[kMaxSmemSegs];
    __shared__ long long clk0;
    __shared__ unsigned long long ns0;
    cg::cluster_group cluster = cg::this_cluster();
    const int S = (int)cluster.num_blocks();
    const int cr = (int)cluster.block_rank();
    const int tid = threadIdx.x, lane = tid & 31;
    const bool lead = cr == 0 && tid == 0;
    const int32_t nw = p.nwords;
    // three truth buffers in rotation: pass k reads v_k from buf(k) and writes v_{k+1} into
    // buf(k+1); the other CTAs' ORs of pass k+1 land in buf(k+2), which nobody reads while
    // pass k's new atoms are counted after the barrier
    auto buf = [&](int i) { return cbuf + (int64_t)i * nw; };
    if (lead) {
        clk0 = clock64();
        ns0 = globaltimer();
        *p.tail_next = 0;
        *p.status_next = 0;
        if (p.stats)
            for (int i = 0; i < 6; ++i) p.stats[i] = 0;
    }
    if (p.nseg <= kMaxSmemSegs)
        for (int32_t s = tid; s < p.nseg; s += blockDim.x) ssegs[s] = p.segs[s];
    const Segment *segs = p.nseg <= kMaxSmemSegs ? ssegs : p.segs;
    // the program planes: staged in shared memory after the truth buffers when they fit
    // (one CTA, small programs: every pass then runs out of shared memory), else read
    // from global memory (L2) each pass
    const int32_t nq = (int32_t)(p.n_slots >> 2);
    const int4 *lb = reinterpret_cast<const int4 *>(p.lead32);
    const int4 *hb = reinterpret_cast<const int4 *>(p.head);
    const int32_t *colg = p.col;
    if (p.stage_planes) {
        int4 *sl = reinterpret_cast<int4 *>(cbuf + 3 * nw);
        int4 *sh = sl + nq;
        int4 *sc = sh + nq;
        const int64_t ncol4 = p.stream_entries >> 2;
        for (int32_t i = tid; i < nq; i += blockDim.x) {
            sl[i] = __ldg(lb + i);
            sh[i] = __ldg(hb + i);
        }
        for (int64_t i = tid; i < ncol4; i += blockDim.x) sc[i] = __ldg(reinterpret_cast<const int4 *>(p.col) + i);
        lb = sl;
        hb = sh;
        colg = reinterpret_cast<const int32_t *>(sc);
    }
    // block-wide sum of one value per thread (the count of new atoms); two barriers
    // block-wide sum of one value per thread into s_cnt[par] (zeroed a pass ahead); one barrier
    auto block_sum = [&](int32_t x, int par) {
        for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
        if (lane == 0 && x) atomicAdd(&s_cnt[par], x);
        __syncthreads();
        return s_cnt[par];
    };
    if (tid == 0) {
        s_cnt[0] = s_cnt[1] = 0;
        s_qn[0] = s_qn[1] = 0;
    }
    __syncthreads();
    // v_0 = (v0 restricted to the original atoms) | facts | ⊤ in both buffers (Def. 4), its
    // size, and the stages of the original atoms (this CTA's words)
    int32_t pc = 0;
    for (int32_t w = tid; w < nw; w += blockDim.x) {
        const int64_t lo = (int64_t)w * 32;
        uint32_t orig = __ldg(p.factbits + w);
        if (p.v0 && w < p.v0_words) {
            uint32_t v = __ldg(p.v0 + w);
            if (lo + 32 > p.n_out) v &= lo >= p.n_out ? 0u : ((1u << (uint32_t)(p.n_out - lo)) - 1u);
            orig |= v;
        }
        if (lo + 32 > p.n) orig &= lo >= p.n ? 0u : ((1u << (uint32_t)(p.n - lo)) - 1u);
        uint32_t bits = orig;
        if (w == (p.top >> 5)) bits |= 1u << (p.top & 31);
        buf(0)[w] = bits;
        buf(1)[w] = bits;
        buf(2)[w] = bits;
        pc += __popc(orig);
        if (p.stage && (w % S) == cr)
            for (int b = 0; b < 32 && lo + b < p.n_out; ++b) p.stage[lo + b] = ((orig >> b) & 1u) ? 0 : -1;
    }
    int32_t total = block_sum(pc, 1);   // (slot 1: pass 0 counts into slot 0)
    cluster.sync();   // (every CTA's buffers initialised before any remote OR)
    if (lead && p.pops && p.pop_cap > 0) p.pops[0] = total;
    const int32_t step = S * (int32_t)blockDim.x;
#define CDBG(k, i) p.dbg[((k) * gridDim.x + blockIdx.x) * 8 + (i)]
    if (p.dbg && tid == 0) CDBG(0, 6) = ns0;
    for (int k = 0;; ++k) {
        uint32_t *rd = buf(k % 3);
        uint32_t *wr = buf((k + 1) % 3);
        if (p.dbg && tid == 0 && k < 16) CDBG(k, 0) = globaltimer();
        if (k > 0)   // wr held v_{k-2}: bring it up to v_k (remote ORs may already arrive)
            for (int32_t w = tid; w < nw; w += blockDim.x) {
                const uint32_t x = rd[w] & ~wr[w];
                if (x) atomicOr(wr + w, x);
            }
        // (the merge's ORs commute with this pass's; s_qn[k & 1] and s_cnt[k & 1] were zeroed
        // during pass k-1, after its stream barrier -- past every reader of pass k-2)
        if (p.dbg && tid == 0 && k < 16) CDBG(k, 1) = globaltimer();
        // LEAD pass over this CTA's quads of the flat planes: a row whose lead atom is in v_k
        // and whose head is not is queued (one reservation per warp and quad step); the
        // queue is verified after the stream with every thread.  A full queue verifies the
        // row at once.  (warp-uniform trip count: the loop body has warp collectives)
        for (int32_t q0 = cr * (int32_t)blockDim.x + tid; q0 - lane < nq; q0 += step * U) {
            int4 a[U], h[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int32_t q = q0 + u * step;
                a[u] = q < nq ? lb[q] : make_int4(p.n_ext_atoms - 1, 0, 0, 0);
                h[u] = q < nq ? hb[q] : make_int4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int32_t q = q0 + u * step;
                const int32_t av[4] = {a[u].x, a[u].y, a[u].z, a[u].w}, hv[4] = {h[u].x, h[u].y, h[u].z, h[u].w};
                unsigned cand = 0;
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    cand |= (q < nq && sm_bit(rd, (uint32_t)av[e]) && !sm_bit(rd, (uint32_t)hv[e])) ? (1u << e) : 0u;
                const unsigned any = __ballot_sync(0xFFFFFFFFu, cand != 0);
                if (!any) continue;
                const int c = __popc(cand);
                int incl = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                    if (lane >= o) incl += y;
                }
                int base = 0;
                if (lane == 31) base = atomicAdd(&s_qn[k & 1], incl);
                base = __shfl_sync(0xFFFFFFFFu, base, 31) + incl - c;
                for (unsigned f = cand; f; f &= f - 1, ++base) {
                    const int32_t slot = q * 4 + __ffs(f) - 1;
                    if (base < kClQueue) cl_q[base] = slot;
                    else cl_verify(p, segs, colg, reinterpret_cast<const int32_t *>(hb), rd, wr, slot);
                }
            }
        }
        __syncthreads();
        if (tid == 0) {   // the next pass's slots (their last readers, in pass k-1, are past this barrier)
            s_qn[(k + 1) & 1] = 0;
            s_cnt[(k + 1) & 1] = 0;
        }
        {
            const int32_t nc = min(s_qn[k & 1], kClQueue);
            for (int32_t i = tid; i < nc; i += blockDim.x)
                cl_verify(p, segs, colg, reinterpret_cast<const int32_t *>(hb), rd, wr, cl_q[i]);
        }
        if (p.dbg && k < 16 && lane == 0) atomicMax(&CDBG(k, 2), globaltimer());
        if (S > 1) {   // this CTA's new bits into every other CTA's v_{k+1}
            __syncthreads();
            for (int32_t w = tid; w < nw; w += blockDim.x) {
                const uint32_t d = wr[w] & ~rd[w];
                if (d)
                    for (int r = 1; r < S; ++r) {
                        const int t = cr + r < S ? cr + r : cr + r - S;
                        atomicOr(cluster.map_shared_rank(wr, t) + w, d);
                    }
            }
        }
        if (S > 1) cluster.sync();
        else __syncthreads();
        if (p.dbg && tid == 0 && k < 16) CDBG(k, 3) = globaltimer();
        // the new atoms of pass k: counted by every CTA over all words (the same complete
        // v_{k+1} everywhere), stages written by each word's owner
        int32_t nn = 0;
        for (int32_t w = tid; w < nw; w += blockDim.x) {
            const uint32_t d = wr[w] & ~rd[w];
            if (!d) continue;
            nn += __popc(d & (w == (p.top >> 5) ? ~(1u << (p.top & 31)) : ~0u));
            if (p.stage && (w % S) == cr)
                for (uint32_t b = d; b;) {
                    const int i = __ffs(b) - 1;
                    b &= b - 1;
                    const int64_t a = (int64_t)w * 32 + i;
                    if (a < p.n_out) p.stage[a] = k + 1;
                }
        }
        const int32_t sum = block_sum(nn, k & 1);
        if (p.dbg && tid == 0 && k < 16) CDBG(k, 5) = globaltimer();
        if (lead && p.stats)
            atomicAdd(p.stats + 0, (p.stage_planes ? 0ull : 8ull * (unsigned long long)p.n_slots) +
                                       4ull * (unsigned long long)sum);
        if (sum == 0 || k + 1 >= p.max_passes || k + 1 == p.user_cap) {
            if (lead) {
                *p.iters_out = k + 1;
                if (sum != 0) atomicOr(p.status_out, k + 1 == p.user_cap ? kStCapped : kStGuard);
                if (p.status_user) *p.status_user = atomicOr(p.status_out, 0);
                if (p.stats) {
                    if (p.stage_planes)   // (the planes were read once, into shared memory)
                        atomicAdd(p.stats + 0, 8ull * (unsigned long long)p.n_slots +
                                                   4ull * (unsigned long long)p.stream_entries);
                    p.stats[1] = (unsigned long long)(k + 1);   // (every pass is a LEAD pass)
                    p.stats[4] = (unsigned long long)(clock64() - clk0);
                    p.stats[5] = globaltimer() - ns0;
                }
            }
            // the model (v_{k+1}, in wr) over the original atoms, this CTA's words
            for (int64_t i = cr * (int64_t)blockDim.x + tid; i < p.out_wn; i += (int64_t)S * blockDim.x) {
                const int64_t w = p.out_w0 + i;
                unsigned long long v = (unsigned long long)wr[2 * w] | ((unsigned long long)wr[2 * w + 1] << 32);
                const int64_t lo = w * 64;
                if (lo + 64 > p.n_out) v &= (1ull << (uint32_t)(p.n_out - lo)) - 1ull;
                p.model_out[i] = v;
            }
            if (p.dbg && tid == 0) CDBG(1, 7) = globaltimer();
            return;   // (no remote access follows the last cluster barrier)
        }
        total += sum;
        if (lead && p.pops && k + 1 < p.pop_cap) p.pops[k + 1] = total;
    }
#undef CDBG
}

// ------------------------------------------------------------------------------------
// least model: ONE CTA, the whole program in shared memory, semi-naive row lists
// ------------------------------------------------------------------------------------
//
// Programs whose rows fit shared memory in 16-bit ids (C1; DESIGN.md "Small-program
// kernel").  lp_load packs the rows (fact heads and always-true body atoms dropped) as
// 8-byte records (head, body range, first body atom), the body ids and the transpose (rows
// by body atom).  Pass 0 evaluates every row against v_0; pass k > 0 only the rows that
// hold an atom derived in pass k-1 (any other row fired before or still misses an atom):
// the same θ(M v_k) per pass as the other kernels -- same model, iters, popcounts, stages.
// A firing row ORs its head into v_{k+1} (the atomic's old value tells the first deriver,
// which lists the head and the rows it occurs in for the next pass); after a block barrier
// the listed heads are ORed into v_k.  Two block barriers per pass, no global traffic in
// the loop apart from the stage stores.
constexpr int kSmallThreads = 768;   // (C1, L2 flushed: 768 0.0171 ms, 1024 0.0190, 512 0.0192, 256 0.0212; LP_SMALL_THREADS)
__global__ void __launch_bounds__(1024, 1) lm_small_kernel(const __grid_constant__ LMParams p) {
    extern __shared__ __align__(16) unsigned long long smb[];
    const int tid = threadIdx.x, lane = tid & 31;
    const int32_t nr = p.sm_nr, nnz = p.sm_nnz, ne = p.n_ext_atoms, nw = p.nwords;
    uint4 *blob = reinterpret_cast<uint4 *>(smb);
    const uint2 *rrec = reinterpret_cast<const uint2 *>(smb);   // (head | begin << 16, end | first body atom << 16)
    const uint16_t *rbody = reinterpret_cast<const uint16_t *>(rrec + nr);
    const uint16_t *optr = rbody + nnz;
    const uint16_t *orow = optr + ne + 1;
    uint32_t *cur = reinterpret_cast<uint32_t *>(smb + 2 * (int64_t)p.sm_blob16);   // v_k
    uint32_t *nxt = cur + nw;                                                       // v_{k+1}
    uint16_t *la = reinterpret_cast<uint16_t *>(nxt + nw);    // [ne] atoms derived in this pass
    uint16_t *lr0 = la + ne + (ne & 1);                       // [nnz] x 2: the rows to evaluate in
    uint16_t *lr1 = lr0 + nnz + (nnz & 1);                    //   this pass / in the next one
    __shared__ int32_t s_na[2], s_nr[2], s_tot;
    __shared__ long long clk0;
    __shared__ unsigned long long ns0;
    if (tid == 0) {
        clk0 = clock64();
        ns0 = globaltimer();
        *p.tail_next = 0;
        *p.status_next = 0;
        if (p.stats)
            for (int i = 0; i < 6; ++i) p.stats[i] = 0;
        s_na[0] = s_na[1] = s_nr[0] = s_nr[1] = 0;
        s_tot = 0;
    }
    for (int32_t i = tid; i < p.sm_blob16; i += blockDim.x) blob[i] = __ldg(p.sm_blob + i);
    __syncthreads();
    // v_0 = (v0 restricted to the original atoms) | facts | ⊤ in both buffers (Def. 4), its
    // size, and the stages of the original atoms
    int32_t pc = 0;
    for (int32_t w = tid; w < nw; w += blockDim.x) {
        const int64_t lo = (int64_t)w * 32;
        uint32_t orig = __ldg(p.factbits + w);
        if (p.v0 && w < p.v0_words) {
            uint32_t x = __ldg(p.v0 + w);
            if (lo + 32 > p.n_out) x &= lo >= p.n_out ? 0u : ((1u << (uint32_t)(p.n_out - lo)) - 1u);
            orig |= x;
        }
        if (lo + 32 > p.n) orig &= lo >= p.n ? 0u : ((1u << (uint32_t)(p.n - lo)) - 1u);
        uint32_t bits = orig;
        if (w == (p.top >> 5)) bits |= 1u << (p.top & 31);
        cur[w] = bits;
        nxt[w] = bits;
        pc += __popc(orig);
        if (p.stage)
            for (int b = 0; b < 32 && lo + b < p.n_out; ++b) p.stage[lo + b] = ((orig >> b) & 1u) ? 0 : -1;
    }
    for (int o = 16; o; o >>= 1) pc += __shfl_xor_sync(0xFFFFFFFFu, pc, o);
    if (lane == 0 && pc) atomicAdd(&s_tot, pc);
    __syncthreads();
    int32_t total = s_tot;
    if (tid == 0 && p.pops && p.pop_cap > 0) p.pops[0] = total;
    for (int k = 0;; ++k) {
        const uint16_t *rows = (k & 1) ? lr1 : lr0;
        uint16_t *lrn = (k & 1) ? lr0 : lr1;
        const int32_t nrow = k == 0 ? nr : s_nr[k & 1];
        for (int32_t i = tid; i < nrow; i += blockDim.x) {
            const uint2 rc = rrec[k == 0 ? i : (int32_t)rows[i]];
            const uint32_t h = rc.x & 0xFFFFu, e = rc.y & 0xFFFFu, b0 = rc.y >> 16;
            bool ok = !sm_bit(cur, h) && (b0 == 0xFFFFu || sm_bit(cur, b0));
            for (uint32_t j = (rc.x >> 16) + 1; j < e && ok; ++j) ok = sm_bit(cur, rbody[j]);
            if (!ok) continue;
            const uint32_t bit = 1u << (h & 31);
            if (atomicOr(nxt + (h >> 5), bit) & bit) continue;   // (another row derived h in this pass)
            if (p.stage && (int32_t)h < p.n_out) p.stage[h] = k + 1;
            const uint32_t o0 = optr[h], o1 = optr[h + 1];
            cg::coalesced_group g = cg::coalesced_threads();
            int32_t base = 0;
            if (g.thread_rank() == 0) base = atomicAdd(&s_na[k & 1], (int32_t)g.size());
            base = g.shfl(base, 0) + (int32_t)g.thread_rank();
            LP_CHECK(h < (uint32_t)ne && base < ne && o1 <= (uint32_t)nnz);
            la[base] = (uint16_t)h;
            if (o1 > o0) {
                const int32_t rpos = atomicAdd(&s_nr[(k + 1) & 1], (int32_t)(o1 - o0));
                LP_CHECK(rpos + (int32_t)(o1 - o0) <= nnz);
                uint16_t *dst = lrn + rpos;
                for (uint32_t o = o0; o < o1; ++o) *dst++ = orow[o];
            }
        }
        __syncthreads();
        const int32_t sum = s_na[k & 1];   // the atoms derived in pass k (⊤ is never a head)
        if (tid == 0 && p.stats)
            atomicAdd(p.stats + 0, 8ull * (unsigned long long)nrow + 4ull * (unsigned long long)sum);
        if (sum == 0 || k + 1 >= p.max_passes || k + 1 == p.user_cap) {
            if (tid == 0) {
                *p.iters_out = k + 1;
                if (sum != 0) atomicOr(p.status_out, k + 1 == p.user_cap ? kStCapped : kStGuard);
                if (p.status_user) *p.status_user = atomicOr(p.status_out, 0);
                if (p.stats) {
                    atomicAdd(p.stats + 0, 16ull * (unsigned long long)p.sm_blob16);   // (the blob, read once)
                    p.stats[1] = (unsigned long long)(k + 1);
                    p.stats[4] = (unsigned long long)(clock64() - clk0);
                    p.stats[5] = globaltimer() - ns0;
                }
            }
            // the model (v_{k+1}) over the original atoms
            for (int64_t i = tid; i < p.out_wn; i += blockDim.x) {
                const int64_t w = p.out_w0 + i;
                unsigned long long x = (unsigned long long)nxt[2 * w] | ((unsigned long long)nxt[2 * w + 1] << 32);
                const int64_t lo = w * 64;
                if (lo + 64 > p.n_out) x &= (1ull << (uint32_t)(p.n_out - lo)) - 1ull;
                p.model_out[i] = x;
            }
            return;
        }
        total += sum;
        if (tid == 0 && p.pops && k + 1 < p.pop_cap) p.pops[k + 1] = total;
        // v_{k+1} into v_k for the derived atoms; the counters of the pass after next
        for (int32_t i = tid; i < sum; i += blockDim.x) {
            const uint32_t h = la[i];
            atomicOr(cur + (h >> 5), 1u << (h & 31));
        }
        if (tid == 0) {
            s_na[(k + 1) & 1] = 0;
            s_nr[k & 1] = 0;
        }
        __syncthreads();
    }
}

cudaError_t launch_lm_small(const LMParams &p, size_t smem, cudaStream_t st, int threads) {
    lm_small_kernel<<<1, threads > 0 ? threads : kSmallThreads, smem, st>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_lm_cluster(const LMParams &p, int cluster, size_t smem, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    const int threads = p.cl_threads > 0 ? p.cl_threads : kThreads;
    cfg.gridDim = dim3((unsigned)cluster);
    cfg.blockDim = dim3((unsigned)threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)cluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if ((p.n_slots >> 2) <= 2LL * cluster * threads) return cudaLaunchKernelEx(&cfg, lm_cluster_kernel<1>, p);
    return cudaLaunchKernelEx(&cfg, lm_cluster_kernel<4>, p);
}

// The largest cluster (<= want) of lm_cluster_kernel that fits with `smem` bytes per CTA.
int lm_cluster_max(int want, size_t smem) {
    // (the attributes are the kernels', shared by every loaded program: set the maximum)
    const void *ks[2] = {(const void *)lm_cluster_kernel<1>, (const void *)lm_cluster_kernel<4>};
    for (const void *k : ks)
        if (cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess ||
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmemBytes) != cudaSuccess) {
            cudaGetLastError();
            return 0;
        }
    for (int c = want; c >= 1; --c) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)c);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)c;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int n1 = 0, n4 = 0;
        if (cudaOccupancyMaxActiveClusters(&n1, ks[0], &cfg) == cudaSuccess && n1 >= 1 &&
            cudaOccupancyMaxActiveClusters(&n4, ks[1], &cfg) == cudaSuccess && n4 >= 1)
            return c;
        cudaGetLastError();
    }
    return 0;
}

// ------------------------------------------------------------------------------------
// stable models: bit-sliced guess matrix, 64 guesses per uint64 word
// ------------------------------------------------------------------------------------

__device__ __forceinline__ unsigned long long valid_word(int64_t w, int32_t W, int64_t G) {
    if (w >= W) return 0ull;
    const int64_t rem = G - w * 64;
    return rem >= 64 ? ~0ull : ((1ull << rem) - 1ull);
}

// bit b of the result = bit i of the guess id 64*w + b
__device__ __forceinline__ unsigned long long count_pattern(int i, int64_t w) {
    switch (i) {
        case 0: return 0xAAAAAAAAAAAAAAAAull;
        case 1: return 0xCCCCCCCCCCCCCCCCull;
        case 2: return 0xF0F0F0F0F0F0F0F0ull;
        case 3: return 0xFF00FF00FF00FF00ull;
        case 4: return 0xFFFF0000FFFF0000ull;
        case 5: return 0xFFFFFFFF00000000ull;
        default: return ((w >> (i - 6)) & 1) ? ~0ull : 0ull;
    }
}

// Initial matrix M_0 (Def. 8): ⊤ and fact rows all ones (over the
// valid guesses), abar rows from the guesses, every other row zero (memset before).
__device__ void st_init_phase(const STParams &p, int64_t gtid, int64_t gthreads) {
    const int64_t rows = 1 + (int64_t)p.nfacts + p.k;
    const int64_t total = rows * p.Wp;
    for (int64_t x = gtid; x < total; x += gthreads) {
        const int64_t r = x / p.Wp, w = x % p.Wp;
        const unsigned long long valid = valid_word(w, p.W, p.G);
        int32_t row;
        unsigned long long v;
        if (r == 0) {
            row = p.top;
            v = valid;
        } else if (r <= p.nfacts) {
            row = p.facts[r - 1];
            v = valid;
        } else {
            const int32_t j = (int32_t)(r - 1 - p.nfacts);
            row = p.negated_ext[j];
            if (p.guesses) {
                v = (w < p.W ? p.guesses[(int64_t)j * p.W + w] : 0ull) & valid;
            } else {
                const int32_t rank = p.free_rank[j];
                v = rank < 0 ? 0ull : (count_pattern(rank, w + p.woff) & valid);   // global word
            }
        }
        p.T0[(int64_t)row * p.Wp + w] = v;
        p.T1[(int64_t)row * p.Wp + w] = v;
        // the row's "true in some guess" bit: one atomic per group of lanes on the same row
        // (a row's Wp words are consecutive x: up to 32 lanes would hit one word)
        const unsigned am = __activemask();
        const unsigned same = __match_any_sync(am, row);
        const bool any = __any_sync(same, v != 0ull);
        if (any && (threadIdx.x & 31) == __ffs(same) - 1) {
            const uint32_t g = (uint32_t)row >> p.any_shift;
            atomicOr(p.any_rw + (g >> 5), 1u << (g & 31));
        }
    }
}

// Zero the matrix rows the previous stable call changed -- exactly the rows with a pass
// tag in mark[] -- in both buffers (rows it did not change are still zero), the tags
// themselves and the call's counters.  A warp per row, lanes over its words.
__device__ void st_clear_phase(const STParams &p, int32_t clear_rows, int64_t gtid, int64_t gthreads) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = gtid >> 5;
    const int64_t nwarps = gthreads >> 5;
    for (int64_t h0 = warp * 32; h0 < p.n_ext; h0 += nwarps * 32) {
        const int64_t h = h0 + lane;
        const bool tagged = h < p.n_ext && __ldcg(p.mark + h) != 0;
        unsigned m = __ballot_sync(0xFFFFFFFFu, tagged);
        if (tagged) p.mark[h] = 0;
        while (m && clear_rows) {
            const int e = __ffs(m) - 1;
            m &= m - 1;
            for (int32_t w = lane; w < p.Wp; w += 32) {
                p.T0[(h0 + e) * p.Wp + w] = 0ull;
                p.T1[(h0 + e) * p.Wp + w] = 0ull;
            }
        }
    }
    for (int64_t w = gtid; w < p.any_words; w += gthreads) {
        p.any_rw[w] = 0u;
        p.gfull[w] = 0u;
    }
    if (gtid == 0) {
        *p.tail = 0;
        p.pcnt[0] = p.pcnt[1] = p.pcnt[2] = 0;
        if (p.lbar) p.lbar[0] = p.lbar[1] = 0ull;   // (the pass barrier words; read after a grid barrier)
        *p.status_out = 0;
        *p.n_accepted = 0;
    }
}

// Algorithm 3's test for every guess word: accept iff a_j ∈ M ⟺ b̄_j ∉ M for every j.
__device__ void st_check_phase(const STParams &p, int64_t gtid, int64_t gthreads) {
    for (int64_t w = gtid; w < p.W; w += gthreads) {
        unsigned long long ok = valid_word(w, p.W, p.G);
        for (int32_t j = 0; j < p.k; ++j)
            ok &= __ldcg(p.T0 + (int64_t)p.negated[j] * p.Wp + w) ^ __ldcg(p.T0 + (int64_t)(p.n_atoms + j) * p.Wp + w);
        p.accepted[w] = ok;
        if (ok) atomicAdd((unsigned long long *)p.n_accepted, (unsigned long long)__popcll(ok));
    }
}

// One candidate AND-row, all guess words: acc = AND of the body rows of T_k; the new
// bits (acc & ~T_k[head]) are ORed into T_{k+1}[head].  A warp owns the row, each lane
// two words (one 16-byte load per body atom).
__device__ __forceinline__ void st_row(const STParams &p, const Segment &sg, int64_t i,
                                       const unsigned long long *rd, unsigned long long *wr,
                                       int k, int lane, int32_t *pc, int32_t base, int32_t *sapp = nullptr) {
    // the head and the first kB body ids in one round trip, then the head row and those body
    // rows in a second one (independent loads in flight), then the new bits of the guesses
    // whose head is still false; positions past kB (long bodies) 4 at a time with the
    // short-circuit
    constexpr int kB = 6;
    const int32_t h = __ldg(p.head + sg.slot_off + i);
    int32_t a0[kB];
#pragma unroll
    for (int j = 0; j < kB; ++j)
        a0[j] = j < sg.L ? __ldg(p.col + sg.col_off + (int64_t)j * sg.count_pad + i) : -1;
    bool changed = false;
    for (int32_t w = 2 * lane; w < p.Wp; w += 64) {
        const ulonglong2 hv = __ldcg(reinterpret_cast<const ulonglong2 *>(rd + (int64_t)h * p.Wp + w));
        ulonglong2 r0[kB];
#pragma unroll
        for (int j = 0; j < kB; ++j)
            r0[j] = a0[j] >= 0 ? __ldcg(reinterpret_cast<const ulonglong2 *>(rd + (int64_t)a0[j] * p.Wp + w))
                               : make_ulonglong2(~0ull, ~0ull);
        ulonglong2 acc = make_ulonglong2(~hv.x, ~hv.y);
#pragma unroll
        for (int j = 0; j < kB; ++j) {
            acc.x &= r0[j].x;
            acc.y &= r0[j].y;
        }
        for (int32_t j0 = kB; j0 < sg.L && (acc.x | acc.y); j0 += 4) {
            int32_t a[4];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                a[j] = j0 + j < sg.L ? __ldg(p.col + sg.col_off + (int64_t)(j0 + j) * sg.count_pad + i) : -1;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (a[j] >= 0) {
                    const ulonglong2 r = __ldcg(reinterpret_cast<const ulonglong2 *>(rd + (int64_t)a[j] * p.Wp + w));
                    acc.x &= r.x;
                    acc.y &= r.y;
                }
        }
        if (acc.x) { atomicOr(wr + (int64_t)h * p.Wp + w, acc.x); changed = true; }
        if (acc.y) { atomicOr(wr + (int64_t)h * p.Wp + w + 1, acc.y); changed = true; }
    }
    if (__any_sync(0xFFFFFFFFu, changed) && lane == 0) {
        if (atomicExch(p.mark + h, k + 1) != k + 1) {
            // this pass's list (ring segment k % 3, its own counter)
            const int32_t pos = atomicAdd(pc, 1);
            if (sapp) atomicAdd(sapp, 1);   // (the CTA's appends: carried by the pass barrier)
            LP_CHECK(pos < p.ring_cap);
            p.order[base + pos] = h;   // (mark[h] != 0 afterwards: the next call clears row h)
        }
    }
}

// st_row for an armed row given by its record o (head, L, body positions 1..5, slot) and
// its lead atom a (body position 0): the same work without the head / body-id loads.
// Bodies longer than 6 go through st_row (the slot's segment).
__device__ __forceinline__ void st_row_rec(const STParams &p, int32_t o, int32_t a,
                                           const unsigned long long *rd, unsigned long long *wr,
                                           int k, int lane, int32_t *pc, int32_t base, int32_t *sapp) {
    const int4 r0 = __ldg(p.arec + 2 * (int64_t)o);
    const int4 r1 = __ldg(p.arec + 2 * (int64_t)o + 1);
    const int32_t h = r0.x, L = r0.y;
    if (L > 6) {
        const int32_t slot = r1.w;
        int lo = 0, hi = p.nseg - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (__ldg(&p.segs[mid].slot_off) <= slot) lo = mid; else hi = mid - 1;
        }
        const Segment sg = p.segs[lo];
        st_row(p, sg, slot - sg.slot_off, rd, wr, k, lane, pc, base, sapp);
        return;
    }
    const int32_t b[6] = {a, L > 1 ? r0.z : -1, L > 2 ? r0.w : -1, L > 3 ? r1.x : -1,
                          L > 4 ? r1.y : -1, L > 5 ? r1.z : -1};
    bool changed = false;
    for (int32_t w = 2 * lane; w < p.Wp; w += 64) {
        const ulonglong2 hv = __ldcg(reinterpret_cast<const ulonglong2 *>(rd + (int64_t)h * p.Wp + w));
        ulonglong2 r[6];
#pragma unroll
        for (int j = 0; j < 6; ++j)
            r[j] = b[j] >= 0 ? __ldcg(reinterpret_cast<const ulonglong2 *>(rd + (int64_t)b[j] * p.Wp + w))
                             : make_ulonglong2(~0ull, ~0ull);
        ulonglong2 acc = make_ulonglong2(~hv.x, ~hv.y);
#pragma unroll
        for (int j = 0; j < 6; ++j) {
            acc.x &= r[j].x;
            acc.y &= r[j].y;
        }
        if (acc.x) { atomicOr(wr + (int64_t)h * p.Wp + w, acc.x); changed = true; }
        if (acc.y) { atomicOr(wr + (int64_t)h * p.Wp + w + 1, acc.y); changed = true; }
    }
    if (__any_sync(0xFFFFFFFFu, changed) && lane == 0) {
        if (atomicExch(p.mark + h, k + 1) != k + 1) {
            const int32_t pos = atomicAdd(pc, 1);
            if (sapp) atomicAdd(sapp, 1);
            LP_CHECK(pos < p.ring_cap);
            p.order[base + pos] = h;
        }
    }
}

// Algorithm 2: M_{k+1} = θ(M_P M_k) over all guess columns at
// once, until no word changes.  Shared memory holds one "any guess" bit per extended
// atom; a row whose body has an atom false in every guess is skipped after the bit
// test, so only candidate rows gather the 8·Wp-byte guess rows.
template <bool CL>
__device__ __forceinline__ void st_run(const STParams &p, int32_t clear_rows) {
    extern __shared__ uint32_t sm[];
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + tid;
    const int64_t gthreads = (int64_t)gridDim.x * blockDim.x;
    const int64_t gwarp = gtid >> 5, nwarps = gthreads >> 5;
    __shared__ uint32_t st_q[kStQueue];  // candidate rows of this CTA's scan: slot | segment << 27
    __shared__ int32_t st_qn, st_qover;
    // armed passes (exact any-filter, records available):
    // the rows whose lead atom is true in some guess and whose head is not true in every
    // guess, as (record, lead) pairs in two shared-memory lists after the filter bits, and
    // this pass's candidates among them
    __shared__ int2 st_qa[kStQueueA];
    __shared__ int32_t sa_n[2], sa_over, sa_qn;
    // (grid launches) the pass barrier carries this CTA's appends: no count read back
    __shared__ int32_t s_st_app, s_st_cnt;
    __shared__ unsigned long long s_st_prev[2];
    int32_t *const sapp = CL ? nullptr : &s_st_app;
    bool armed = p.arec != nullptr && p.any_shift == 0;
    int acur = 0;
    int2 *const alist = reinterpret_cast<int2 *>(sm + p.any_words * (p.use_full ? 2 : 1));
    if (threadIdx.x == 0) {
        sa_n[0] = sa_n[1] = 0;
        sa_over = 0;
        sa_qn = 0;
        s_st_app = 0;
        s_st_prev[0] = s_st_prev[1] = 0ull;
    }
    // CTA b owns the records [b * arm_cap, (b + 1) * arm_cap) (the host sizes arm_cap so the
    // grid covers all of them): an atom that became true in some guess arms the part of its
    // record range this CTA owns, so a list never holds more than arm_cap entries
    const int32_t own_lo = (int32_t)blockIdx.x * p.arm_cap, own_hi = own_lo + p.arm_cap;
    auto st_arm = [&](int32_t a) {
        const int32_t lo = max(__ldg(p.arm_ptr + a), own_lo), hi = min(__ldg(p.arm_ptr + a + 1), own_hi);
        if (hi <= lo) return;
        int32_t pos = atomicAdd(&sa_n[acur], hi - lo);
        LP_CHECK(pos + (hi - lo) <= p.arm_cap);
        for (int32_t o = lo; o < hi; ++o) alist[(int64_t)acur * p.arm_cap + pos++] = make_int2(o, a);
    };
    // the call's set-up, in the same launch: the previous call's rows and this call's
    // counters cleared, then T_0 (Def. 8) and its "any" bits
    const bool dlead = p.dbg && blockIdx.x == 0 && threadIdx.x == 0;   // (phase stamps: dbg[252..255])
    if (dlead) p.dbg[252] = globaltimer();
    st_clear_phase(p, clear_rows, gtid, gthreads);
    pass_barrier<CL>();
    if (dlead) p.dbg[253] = globaltimer();
    st_init_phase(p, gtid, gthreads);
    pass_barrier<CL>();
    if (dlead) p.dbg[254] = globaltimer();
    // shared memory: "true in some guess" bits, then (exact filter only) "true in every
    // guess" bits -- a row whose head is full can change nothing
    uint32_t *full = sm + p.any_words;
    const bool use_full = p.use_full;
    for (int32_t w = tid; w < p.any_words; w += blockDim.x) {
        sm[w] = __ldcg(p.any_init + w);
        if (use_full) full[w] = 0u;
    }
    __syncthreads();
    if (armed) {   // pass 0: the atoms true in some guess of T_0 (⊤, the facts, the guessed abar_j)
        const int32_t rows = 1 + p.nfacts + p.k;
        for (int32_t r = tid; r < rows; r += blockDim.x) {
            const int32_t a = r == 0 ? p.top : r <= p.nfacts ? p.facts[r - 1] : p.negated_ext[r - 1 - p.nfacts];
            if (sm_bit(sm, (uint32_t)a)) st_arm(a);
        }
        __syncthreads();
    }
    // rows changed in pass k-1 and in pass k-2: counts, their lists in ring segments
    // (k-1) % 3 and (k-2) % 3 of p.order (pass k appends to segment k % 3)
    int32_t n1 = 0, n2 = 0;
    constexpr int kStSpec = 2;
    int32_t s1[kStSpec] = {-1, -1}, s2[kStSpec] = {-1, -1};   // this thread's first entries of both lists
    uint32_t fwc[kStSpec] = {0u, 0u};                          // gfull words of s2 (loaded early)
    for (int k = 0;; ++k) {
        const unsigned long long *rd = (k & 1) ? p.T1 : p.T0;
        unsigned long long *wr = (k & 1) ? p.T0 : p.T1;
        const int32_t *l1 = p.order + (int64_t)((k + 2) % 3) * p.ring_cap;   // changed in pass k-1
        if (k > 0) {
            const int32_t *l2 = p.order + (int64_t)((k + 1) % 3) * p.ring_cap;
            // (the first kStSpec x blockDim entries of both lists are in registers: loaded
            // with the count after the barrier)
            // (armed: an atom whose bit was not set yet became true in some guess in pass
            // k-1 -- every CTA sees the same, each arms the records of it that it owns)
            for (int u = 0; u < kStSpec; ++u)
                if (s1[u] >= 0) {
                    const uint32_t g = (uint32_t)s1[u] >> p.any_shift;
                    const uint32_t old = atomicOr(sm + (g >> 5), 1u << (g & 31));
                    if (armed && !((old >> (g & 31)) & 1u)) st_arm(s1[u]);
                }
            for (int64_t i = tid + kStSpec * blockDim.x; i < n1; i += blockDim.x) {
                const int32_t a = __ldcg(l1 + i);
                const uint32_t g = (uint32_t)a >> p.any_shift;
                const uint32_t old = atomicOr(sm + (g >> 5), 1u << (g & 31));
                if (armed && !((old >> (g & 31)) & 1u)) st_arm(a);
            }
            if (use_full) {   // the full marks made during pass k-1 (rows changed in pass k-2)
                // (their gfull words were loaded right after the barrier, beside the list)
                for (int u = 0; u < kStSpec; ++u)
                    if (s2[u] >= 0 && ((fwc[u] >> (s2[u] & 31)) & 1u)) atomicOr(full + (s2[u] >> 5), 1u << (s2[u] & 31));
                for (int64_t i = tid + kStSpec * blockDim.x; i < n2; i += blockDim.x) {
                    const uint32_t h = (uint32_t)__ldcg(l2 + i);
                    if ((__ldcg(p.gfull + (h >> 5)) >> (h & 31)) & 1u) atomicOr(full + (h >> 5), 1u << (h & 31));
                }
            }
            __syncthreads();
        }
        if (tid == 0) {
            st_qn = 0;
            st_qover = 0;
        }
        __syncthreads();
        if (p.dbg && tid == 0 && k < 64) atomicMax(p.dbg + 4 * k + 2, globaltimer());   // pass top done
        if (blockIdx.x == 0 && tid == 0) p.pcnt[(k + 1) % 3] = 0;   // next pass's counter
        if (armed) {
            // armed pass: every listed row is tested from its record -- its head not true in
            // every guess (else dropped for good), its other body atoms true in some guess
            // (then it is a candidate this pass) -- and kept; candidates are processed by
            // every warp of the CTA like the scan's
            const int32_t na = sa_n[acur];
            const int2 *L0 = alist + (int64_t)acur * p.arm_cap;
            int2 *L1 = alist + (int64_t)(acur ^ 1) * p.arm_cap;
            for (int32_t i0 = tid - lane; i0 < na; i0 += blockDim.x) {   // (warp-uniform)
                const int32_t i = i0 + lane;
                int2 e = make_int2(-1, -1);
                bool cand = false;
                if (i < na) {
                    e = L0[i];
                    const int4 r0 = __ldg(p.arec + 2 * (int64_t)e.x);
                    const int4 r1 = __ldg(p.arec + 2 * (int64_t)e.x + 1);
                    const int32_t h = r0.x, L = r0.y;
                    if (!(use_full && sm_bit(full, (uint32_t)h))) {
                        L1[atomicAdd(&sa_n[acur ^ 1], 1)] = e;   // (kept: < na entries)
                        const int32_t b[5] = {r0.z, r0.w, r1.x, r1.y, r1.z};
                        cand = true;
#pragma unroll
                        for (int j = 0; j < 5; ++j) cand = cand && (j + 1 >= L || sm_bit(sm, (uint32_t)b[j]));
                        if (cand && L > 6) {   // positions 6.. from the column planes
                            const int32_t slot = r1.w;
                            int lo = 0, hi = p.nseg - 1;
                            while (lo < hi) {
                                const int mid = (lo + hi + 1) >> 1;
                                if (__ldg(&p.segs[mid].slot_off) <= slot) lo = mid; else hi = mid - 1;
                            }
                            const Segment sg = p.segs[lo];
                            for (int32_t j = 6; j < L && cand; ++j)
                                cand = sm_bit(sm, (uint32_t)__ldg(p.col + sg.col_off + (int64_t)j * sg.count_pad + (slot - sg.slot_off)));
                        }
                    }
                }
                if (p.dbg && cand) atomicAdd(p.dbg + 4 * (k & 63) + 1, 1ull);
                bool over = false;
                if (cand) {
                    const int32_t pos = atomicAdd(&sa_qn, 1);
                    if (pos < kStQueueA) st_qa[pos] = e;
                    else over = true;
                }
                unsigned m = __ballot_sync(0xFFFFFFFFu, over);   // (rare) a full queue: this warp
                while (m) {                                      // processes them itself
                    const int l = __ffs(m) - 1;
                    m &= m - 1;
                    const int32_t o = __shfl_sync(0xFFFFFFFFu, e.x, l), a = __shfl_sync(0xFFFFFFFFu, e.y, l);
                    st_row_rec(p, o, a, rd, wr, k, lane, p.pcnt + k % 3, (k % 3) * p.ring_cap, sapp);
                }
            }
            __syncthreads();
            const int32_t nq_c = min(sa_qn, kStQueueA);
            for (int32_t i = tid >> 5; i < nq_c; i += blockDim.x >> 5) {
                const int2 e = st_qa[i];
                st_row_rec(p, e.x, e.y, rd, wr, k, lane, p.pcnt + k % 3, (k % 3) * p.ring_cap, sapp);
            }
            __syncthreads();   // (the list counters: reset for the next pass)
            if (tid == 0) {
                sa_n[acur] = 0;
                sa_qn = 0;
            }
            acur ^= 1;
        }
        // candidate scan: a lane tests 4 rows (one 16-byte load per body position, lead
        // position first -- usually an atom that is true in no guess -- and the heads
        // against the "full" bits); the warp then processes the candidates one by one.
        // With the flat lead plane (exact mode) one loop covers every segment.
        if (!armed && p.lead32) {
            const int64_t nq = p.n_slots >> 2;
            const int4 *lb = reinterpret_cast<const int4 *>(p.lead32);
            const int4 *hb = reinterpret_cast<const int4 *>(p.head);
            for (int64_t q0 = gwarp * 32; q0 < nq; q0 += nwarps * 32) {
                const int64_t q = q0 + lane;
                unsigned alive = 0;
                int sgi = 0;
                if (q < nq) {
                    const int4 a = ld_stream(lb + q);
                    alive = (sm_bit(sm, (uint32_t)a.x) ? 1u : 0u) | (sm_bit(sm, (uint32_t)a.y) ? 2u : 0u) |
                            (sm_bit(sm, (uint32_t)a.z) ? 4u : 0u) | (sm_bit(sm, (uint32_t)a.w) ? 8u : 0u);
                    if (alive && use_full) {
                        const int4 h = ld_stream(hb + q);
                        alive &= (sm_bit(full, (uint32_t)h.x) ? 0u : 1u) | (sm_bit(full, (uint32_t)h.y) ? 0u : 2u) |
                                 (sm_bit(full, (uint32_t)h.z) ? 0u : 4u) | (sm_bit(full, (uint32_t)h.w) ? 0u : 8u);
                    }
                    if (alive) {   // the quad's segment (quads never straddle segments here)
                        int lo = 0, hi = p.nseg - 1;
                        while (lo < hi) {
                            const int mid = (lo + hi + 1) >> 1;
                            if (__ldg(&p.segs[mid].slot_off) <= q * 4) lo = mid; else hi = mid - 1;
                        }
                        sgi = lo;
                        const int32_t L = __ldg(&p.segs[lo].L);
                        const int64_t cpq = __ldg(&p.segs[lo].count_pad) >> 2;
                        const int4 *cb = reinterpret_cast<const int4 *>(p.col + __ldg(&p.segs[lo].col_off)) +
                                         (q - (__ldg(&p.segs[lo].slot_off) >> 2));
                        for (int32_t j = 1; j < L && alive; ++j) {
                            const int4 c = ld_stream(cb + (int64_t)j * cpq);
                            alive &= (sm_bit(sm, (uint32_t)c.x) ? 1u : 0u) | (sm_bit(sm, (uint32_t)c.y) ? 2u : 0u) |
                                     (sm_bit(sm, (uint32_t)c.z) ? 4u : 0u) | (sm_bit(sm, (uint32_t)c.w) ? 8u : 0u);
                        }
                    }
                }
                if (p.dbg && alive) atomicAdd(p.dbg + 4 * (k & 63) + 1, (unsigned long long)__popc(alive));
                // candidates go to the CTA's shared queue (slot | segment << 27) so that all
                // warps share them; a full queue is drained by the finding warp itself
                for (unsigned f = alive; f && p.cta_queue; f &= f - 1) {
                    const int e = __ffs(f) - 1;
                    const int32_t pos = atomicAdd(&st_qn, 1);
                    if (pos < kStQueue) st_q[pos] = (uint32_t)(q * 4 + e) | ((uint32_t)sgi << 27);
                    else atomicAdd(&st_qover, 1);
                }
                if (!p.cta_queue && alive) st_qover = 1;   // (huge programs: the direct path)
                if (__any_sync(0xFFFFFFFFu, st_qover != 0)) {   // (rare) overflow: old path
                    for (int e = 0; e < 4; ++e) {
                        unsigned m = __ballot_sync(0xFFFFFFFFu, (alive >> e) & 1u);
                        while (m) {
                            const int l = __ffs(m) - 1;
                            m &= m - 1;
                            const int s = __shfl_sync(0xFFFFFFFFu, sgi, l);
                            const Segment sg = p.segs[s];
                            st_row(p, sg, (q0 + l) * 4 + e - sg.slot_off, rd, wr, k, lane, p.pcnt + k % 3,
                                   (k % 3) * p.ring_cap, sapp);
                        }
                    }
                }
            }
            __syncthreads();
            // every warp takes candidates from the shared queue
            const int32_t nq_c = min(st_qn, kStQueue);
            for (int32_t i = tid >> 5; i < nq_c && p.cta_queue; i += blockDim.x >> 5) {
                const uint32_t ent = st_q[i];
                const Segment sg = p.segs[ent >> 27];
                st_row(p, sg, (int64_t)(ent & 0x7FFFFFFu) - sg.slot_off, rd, wr, k, lane, p.pcnt + k % 3,
                       (k % 3) * p.ring_cap, sapp);
            }
        }
        int64_t off = 0;  // rotate each segment's first warp (see all_segments)
        for (int32_t s = 0; s < ((armed || p.lead32) ? 0 : p.nseg); ++s) {
            const Segment sg = p.segs[s];
            const int64_t nq = sg.count_pad >> 2;
            const int64_t gw = gwarp >= off ? gwarp - off : gwarp - off + nwarps;
            off = (off + (nq + 31) / 32) % nwarps;
            const int4 *cb = reinterpret_cast<const int4 *>(p.col + sg.col_off);
            const int4 *hb = reinterpret_cast<const int4 *>(p.head + sg.slot_off);
            for (int64_t q0 = gw * 32; q0 < nq; q0 += nwarps * 32) {
                const int64_t q = q0 + lane;
                unsigned alive = 0;
                if (q < nq) {
                    const int4 a = ld_stream(cb + q);
                    alive = (sm_bit(sm, (uint32_t)a.x >> p.any_shift) ? 1u : 0u) |
                            (sm_bit(sm, (uint32_t)a.y >> p.any_shift) ? 2u : 0u) |
                            (sm_bit(sm, (uint32_t)a.z >> p.any_shift) ? 4u : 0u) |
                            (sm_bit(sm, (uint32_t)a.w >> p.any_shift) ? 8u : 0u);
                    if (alive && use_full) {
                        const int4 h = ld_stream(hb + q);
                        alive &= (sm_bit(full, (uint32_t)h.x) ? 0u : 1u) | (sm_bit(full, (uint32_t)h.y) ? 0u : 2u) |
                                 (sm_bit(full, (uint32_t)h.z) ? 0u : 4u) | (sm_bit(full, (uint32_t)h.w) ? 0u : 8u);
                    }
                    for (int32_t j = 1; j < sg.L && alive; ++j) {
                        const int4 c = ld_stream(cb + (int64_t)j * nq + q);
                        alive &= (sm_bit(sm, (uint32_t)c.x >> p.any_shift) ? 1u : 0u) |
                                 (sm_bit(sm, (uint32_t)c.y >> p.any_shift) ? 2u : 0u) |
                                 (sm_bit(sm, (uint32_t)c.z >> p.any_shift) ? 4u : 0u) |
                                 (sm_bit(sm, (uint32_t)c.w >> p.any_shift) ? 8u : 0u);
                    }
                }
                if (p.dbg && alive) atomicAdd(p.dbg + 4 * (k & 63) + 1, (unsigned long long)__popc(alive));
                for (int e = 0; e < 4; ++e) {
                    unsigned m = __ballot_sync(0xFFFFFFFFu, (alive >> e) & 1u);
                    while (m) {
                        const int l = __ffs(m) - 1;
                        m &= m - 1;
                        st_row(p, sg, (q0 + l) * 4 + e, rd, wr, k, lane, p.pcnt + k % 3, (k % 3) * p.ring_cap, sapp);
                    }
                }
            }
        }
        if (k > 0) {
            // rows changed in pass k-1: copy T_k's words into the other buffer (a warp per
            // row; ORs commute with this pass's, so it only has to finish before the
            // barrier) and mark the rows that are now true in every guess (global, read by
            // every CTA one pass later)
            for (int64_t i = gwarp; i < n1; i += nwarps) {
                const int32_t h = __ldcg(l1 + i);
                bool all1 = true;
                for (int32_t w = lane; w < p.Wp; w += 32) {
                    const int64_t off = (int64_t)h * p.Wp + w;
                    const unsigned long long v = __ldcg(rd + off);
                    if (v != __ldcg(wr + off)) atomicOr(wr + off, v);
                    const unsigned long long valid = valid_word(w, p.W, p.G);
                    all1 = all1 && ((v & valid) == valid);
                }
                if (use_full && __all_sync(0xFFFFFFFFu, all1) && lane == 0)
                    atomicOr(p.gfull + (h >> 5), 1u << (h & 31));
            }
        }
        if (p.dbg && k < 64) {
            __syncthreads();
            if (tid == 0) atomicMax(p.dbg + 4 * k + 3, globaltimer());     // CTA's scan done
        }
        if constexpr (CL) {
            pass_barrier<CL>();
        } else {
            // one 64-bit release-reduction per CTA on the word of this pass's parity:
            // [arrivals:24 | - | appends:32], both growing within a call (differences to the
            // word's last value are this pass's); polled with acquire
            __syncthreads();
            if (tid == 0) {
                const unsigned long long add = (1ull << 40) | (unsigned long long)(uint32_t)s_st_app;
                asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p.lbar + (k & 1)), "l"(add) : "memory");
                const uint32_t target = (uint32_t)((((unsigned long long)(k / 2) + 1ull) * gridDim.x) & 0xFFFFFFull);
                unsigned long long v;
                for (;;) {
                    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p.lbar + (k & 1)) : "memory");
                    if ((((uint32_t)(v >> 40) - target) & 0xFFFFFFu) < 0x800000u) break;
                }
                s_st_cnt = (int32_t)((uint32_t)v - (uint32_t)s_st_prev[k & 1]);
                s_st_prev[k & 1] = v;
                s_st_app = 0;
            }
            __syncthreads();
        }
        // rows changed in this pass: its own counter slot (the next pass appends to
        // another one, so every CTA reads the same value after the barrier); this
        // thread's first entries of the list are loaded together with it (slots past the
        // count hold stale entries of an earlier pass and are dropped)
        int32_t nx[kStSpec];
        uint32_t fwn[kStSpec];   // the gfull words of the rows changed in pass k-1 (marked during pass k)
        for (int u = 0; u < kStSpec; ++u) {
            const int64_t i = tid + (int64_t)u * blockDim.x;
            nx[u] = i < p.ring_cap ? __ldcg(p.order + (int64_t)(k % 3) * p.ring_cap + i) : -1;
            fwn[u] = (use_full && s1[u] >= 0) ? __ldcg(p.gfull + (s1[u] >> 5)) : 0u;
        }
        const int32_t cnt = CL ? cta_pass_counts(p.pcnt + k % 3, nullptr, nullptr).appended : s_st_cnt;
        const bool lead = blockIdx.x == 0 && tid == 0;
        if (p.dbg && lead && k < 64) p.dbg[4 * k] = globaltimer();   // profiling hook
        if (cnt == 0) {
            if (lead) { *p.passes_out = k + 1; }
            break;
        }
        if (k + 1 >= p.max_passes) {
            if (lead) { *p.passes_out = k + 1; atomicOr(p.status_out, kStGuard); }
            break;
        }
        n2 = n1;
        n1 = cnt;
        for (int u = 0; u < kStSpec; ++u) {
            s2[u] = s1[u];
            fwc[u] = fwn[u];
            s1[u] = tid + u * (int)blockDim.x < cnt ? nx[u] : -1;
        }
    }
    // both buffers hold the fixpoint (rows changed in the last pass were copied during it)
    if (dlead) p.dbg[255] = globaltimer();
    st_check_phase(p, gtid, gthreads);
}

template <bool CL>
__global__ void __launch_bounds__(kThreads, 1) st_fixpoint_kernel(const __grid_constant__ STParams p) {
    st_run<CL>(p, p.clear_rows);
    if (blockIdx.x == 0 && threadIdx.x == 0 && p.status_user)
        *p.status_user = *(volatile int32_t *)p.status_out;
}

// ------------------------------------------------------------------------------------
// stable models: compact kernel (the live sub-program in shared memory, a CTA per guess word)
// ------------------------------------------------------------------------------------
//
// The guess columns of Algorithm 2 never interact: M_{k+1} = θ(M_P M_k)
// acts on every column by itself.  A row of M_P can fire in SOME guess only if its whole body
// lies in A*, the least model of P+ with every abar_j true (P+ is definite, so A* contains
// every guess's model); lp_load computes A* once per program and keeps the live rows (body
// ⊆ A*, head not a fact) in compact ids, with their transpose.  When that fits shared
// memory, CTA w runs the whole Jacobi fixpoint of guess word w (64 columns) out of shared
// memory -- block barriers only: no grid barrier, no global traffic inside the loop.  Pass 0
// evaluates every live row; pass k > 0 only the rows with a body atom whose word changed in
// pass k-1 (any other row computes the bits it computed before, already in its head).  The
// CTA then stores its column of the fixpoint matrix over A* (rows outside A* are zero) into
// the compact matrix C[w][A*] (lp_stable_matrix / lp_guess_model expand it), tests Algorithm
// 3's condition and records the word's pass count; the last CTA to
// finish reduces the accepted count and the pass count (max over words = the batched loop's
// passes: a pass changes the matrix iff it changes some column).  Same T_k at every k as
// the batched kernel: same matrix, accepted ids and passes (DESIGN.md "Compact stable
// kernel").
// The CTA's shared memory: the blob (uint16 units: row records[nr][4] (head, body begin, body
// end, first body atom or 0xFFFF for an empty body) | body[nnz] | occ_ptr[na+1] | occ
// row[nnz] | init[na] | pass-0 rows[n0]), then the two column buffers, the change lists and
// their bitmap.  A CTA works on HALF a guess word (32 columns, uint32 columns): twice the
// CTAs and half the column bytes of a whole word.  The atoms that are all ones from T_0 on
// (⊤, the facts) are not among the compact atoms: they never mask a bit and never change.
constexpr uint32_t kCpNone = 0xFFFFu;
struct CpView {
    int32_t na, nr, nnz;
    uint4 *blob;
    const uint2 *rrec;       // (head | begin << 16, end | first body atom << 16)
    const uint16_t *rbody, *optr, *orow, *row0;
    const int16_t *ainit;    // -1: zero in T_0, j >= 0: abar_j
    uint32_t *cur, *nxt;
    uint16_t *la;            // [na] rows of T changed in this pass
    uint16_t *lr0, *lr1;     // [nnz] x 2: the AND-rows to evaluate in this pass / in the next one
    int32_t *s_na, *s_nr;    // [2] each: list counters by pass parity
};

__device__ __forceinline__ CpView cp_view(const STParams &p, unsigned long long *cpb, int32_t *s_cnt) {
    CpView v;
    v.na = p.cp_na;
    v.nr = p.cp_nr;
    v.nnz = p.cp_nnz;
    v.blob = reinterpret_cast<uint4 *>(cpb);
    v.rrec = reinterpret_cast<const uint2 *>(cpb);
    v.rbody = reinterpret_cast<const uint16_t *>(v.rrec + v.nr);
    v.optr = v.rbody + v.nnz;
    v.orow = v.optr + v.na + 1;
    v.ainit = reinterpret_cast<const int16_t *>(v.orow + v.nnz);
    v.row0 = reinterpret_cast<const uint16_t *>(v.ainit + v.na);
    v.cur = reinterpret_cast<uint32_t *>(cpb + 2 * (int64_t)p.cp_blob16);
    v.nxt = v.cur + v.na;
    v.la = reinterpret_cast<uint16_t *>(v.nxt + v.na);
    v.lr0 = v.la + v.na + (v.na & 1);
    v.lr1 = v.lr0 + v.nnz + (v.nnz & 1);
    v.s_na = s_cnt;
    v.s_nr = s_cnt + 2;
    return v;
}

// the blob into shared memory, the list state cleared (ends with a block barrier)
__device__ __forceinline__ void cp_stage(const STParams &p, const CpView &v) {
    const int tid = threadIdx.x;
    for (int32_t i = tid; i < p.cp_blob16; i += blockDim.x) v.blob[i] = __ldg(p.cp_blob + i);
    if (tid == 0) v.s_na[0] = v.s_na[1] = v.s_nr[0] = v.s_nr[1] = 0;
    __syncthreads();
}

// the valid columns of half-word hw (columns 32 hw .. 32 hw + 31)
__device__ __forceinline__ uint32_t valid_half(const STParams &p, int32_t hw) {
    return (uint32_t)(valid_word(hw >> 1, p.W, p.G) >> (32 * (hw & 1)));
}

// The whole Jacobi fixpoint of half-word hw in shared memory; returns its pass count and
// leaves the fixpoint column over A* in v.cur.  cols: the caller's guesses [k][W] (NULL:
// binary counting); SEARCH: they were written by this kernel (no read-only loads).
template <bool SEARCH>
__device__ __forceinline__ int32_t cp_word(const STParams &p, const CpView &v, int32_t hw,
                                           const unsigned long long *cols, bool dl) {
    const int tid = threadIdx.x;
    const int32_t na = v.na;
    uint32_t *cur = v.cur, *nxt = v.nxt;
    const uint32_t valid = valid_half(p, hw);
    const uint32_t *c32 = reinterpret_cast<const uint32_t *>(cols);
    // T_0 (Def. 8) on A* minus the all-ones rows: abar_j from the guesses
    for (int32_t a = tid; a < na; a += blockDim.x) {
        const int32_t ini = v.ainit[a];
        uint32_t x = 0u;
        if (ini >= 0) {
            if (cols) x = (SEARCH ? __ldcg(c32 + (int64_t)ini * 2 * p.W + hw) : __ldg(c32 + (int64_t)ini * 2 * p.W + hw)) & valid;
            else {
                const int32_t rank = __ldg(p.free_rank + ini);
                x = rank < 0 ? 0u : ((uint32_t)(count_pattern(rank, (hw >> 1) + p.woff) >> (32 * (hw & 1))) & valid);
            }
        }
        cur[a] = x;
        nxt[a] = x;
    }
    __syncthreads();
    if (dl) p.dbg[1] = globaltimer();
    // one AND-row against T_k (cur): its new bits are ORed into T_{k+1} (nxt); at its
    // head's first change in this pass the head goes onto the pass's change list (one
    // counter atomic per group of converged lanes) and the rows it occurs in onto the
    // next pass's row list (a row listed twice is evaluated twice: ORs are idempotent)
    auto eval_row = [&](int32_t r, int k) {
        const uint2 rc = v.rrec[r];
        const uint32_t h = rc.x & 0xFFFFu, e = rc.y & 0xFFFFu, b0 = rc.y >> 16;
        const uint32_t ch = cur[h];
        uint32_t acc = valid & ~ch;
        if (b0 != kCpNone) acc &= cur[b0];
        for (uint32_t i = (rc.x >> 16) + 1; i < e && acc; ++i) acc &= cur[v.rbody[i]];
        if (!acc) return;
        // (T_{k+1}[h] = T_k[h] until the pass's first OR, which adds bits T_k[h] lacks: the old
        // value names the first row to change h in this pass)
        if (atomicOr(nxt + h, acc) != ch) return;
        const uint32_t o0 = v.optr[h], o1 = v.optr[h + 1];
        cg::coalesced_group g = cg::coalesced_threads();
        int32_t base = 0;
        if (g.thread_rank() == 0) base = atomicAdd(&v.s_na[k & 1], (int32_t)g.size());
        base = g.shfl(base, 0) + (int32_t)g.thread_rank();
        LP_CHECK(h < (uint32_t)v.na && base < v.na && o1 <= (uint32_t)v.nnz);
        v.la[base] = (uint16_t)h;
        if (o1 > o0) {
            const int32_t rpos = atomicAdd(&v.s_nr[(k + 1) & 1], (int32_t)(o1 - o0));
            LP_CHECK(rpos + (int32_t)(o1 - o0) <= v.nnz);
            uint16_t *dst = ((k & 1) ? v.lr0 : v.lr1) + rpos;
            for (uint32_t o = o0; o < o1; ++o) *dst++ = v.orow[o];
        }
    };
    int32_t passes = 0;
    for (int k = 0;; ++k) {
        // pass 0: the rows whose body lies in T_0's possible atoms (the others hold an atom
        // that is zero in every column of T_0); pass k: the rows with a body atom that
        // changed in pass k-1 (any other row computes the bits it computed before,
        // already in its head)
        const uint16_t *rows = k == 0 ? v.row0 : ((k & 1) ? v.lr1 : v.lr0);
        const int32_t nrow = k == 0 ? p.cp_n0 : v.s_nr[k & 1];
        for (int32_t i = tid; i < nrow; i += blockDim.x) eval_row(rows[i], k);
        __syncthreads();
        ++passes;
        const int32_t nn = v.s_na[k & 1];
        if (dl && k < 60) {
            p.dbg[8 + 2 * k] = globaltimer();
            p.dbg[9 + 2 * k] = (unsigned long long)nrow;
        }
        if (nn == 0) break;   // u = v in every column of the half-word
        // T_{k+1} for the changed rows; the bitmap and the counters of the pass after next
        for (int32_t i = tid; i < nn; i += blockDim.x) {
            const uint32_t h = v.la[i];
            cur[h] = nxt[h];
        }
        if (tid == 0) {
            v.s_na[(k + 1) & 1] = 0;
            v.s_nr[k & 1] = 0;
        }
        __syncthreads();
    }
    if (dl) p.dbg[2] = globaltimer();
    return passes;
}

// a compact id's column bits: -1 = not in A* (never true), -2 = a fact (all ones)
__device__ __forceinline__ uint32_t cp_bits(const CpView &v, int32_t c, uint32_t valid) {
    return c >= 0 ? v.cur[c] : c == -2 ? valid : 0u;
}

// Algorithm 3 on the half-word's fixpoint column (warp 0; every lane
// returns the accepted mask): a_j ∈ M ⟺ abar_j ∉ M for every j
__device__ __forceinline__ uint32_t cp_check(const STParams &p, const CpView &v, int32_t hw,
                                             int32_t cneg, int32_t cabar) {
    const int lane = threadIdx.x & 31;
    const uint32_t valid = valid_half(p, hw);
    uint32_t ok = valid;
    for (int32_t j = lane; j < p.k; j += 32) {
        const int32_t ca = j < 32 ? cneg : __ldg(p.cp_neg + j), cb = j < 32 ? cabar : __ldg(p.cp_abar + j);
        ok &= cp_bits(v, ca, valid) ^ cp_bits(v, cb, valid);
    }
    for (int o = 16; o; o >>= 1) ok &= __shfl_xor_sync(0xFFFFFFFFu, ok, o);
    return ok;
}

__global__ void __launch_bounds__(kThreads, 1) st_compact_kernel(const __grid_constant__ STParams p) {
    extern __shared__ __align__(16) unsigned long long cpb[];
    const int tid = threadIdx.x, lane = tid & 31;
    __shared__ int32_t s_cnt[4], s_last, s_mp;
    __shared__ unsigned long long s_n;
    const CpView v = cp_view(p, cpb, s_cnt);
    const int32_t na = v.na;
    const bool dl = p.dbg && blockIdx.x == 0 && tid == 0;   // (phase stamps: tools/dbg_compact.py)
    if (dl) p.dbg[0] = globaltimer();
    // (Algorithm 3's pairs, compact ids: requested now, used after the fixpoint)
    int32_t cneg = -1, cabar = -1;
    if (tid < 32 && lane < p.k) {
        cneg = __ldg(p.cp_neg + lane);
        cabar = __ldg(p.cp_abar + lane);
    }
    cp_stage(p, v);
    uint32_t *C32 = reinterpret_cast<uint32_t *>(p.cp_C);
    uint32_t *acc32 = reinterpret_cast<uint32_t *>(p.accepted);
    for (int32_t hw = blockIdx.x; hw < 2 * p.W; hw += gridDim.x) {
        const int32_t passes = cp_word<false>(p, v, hw, p.guesses, dl);
        // the half-word's column of the fixpoint matrix over A* (cur = nxt at the fixpoint)
        for (int32_t a = tid; a < na; a += blockDim.x) C32[(int64_t)hw * na + a] = v.cur[a];
        if (tid < 32) {
            const uint32_t ok = cp_check(p, v, hw, cneg, cabar);
            if (lane == 0) {
                acc32[hw] = ok;
                p.cp_pw[hw] = passes;
            }
        }
        if (tid == 0) s_cnt[0] = s_cnt[1] = s_cnt[2] = s_cnt[3] = 0;
        __syncthreads();   // (cur and the counters are rebuilt for the CTA's next half-word)
        if (dl) p.dbg[3] = globaltimer();
    }
    // the last CTA to finish reduces the per-half-word results (fence + ticket)
    if (tid == 0) {
        s_mp = 0;
        s_n = 0ull;
        __threadfence();
        s_last = atomicAdd(p.cp_done, 1) == (int32_t)gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    long long n = 0;
    int32_t mp = 0;
    for (int32_t hw = tid; hw < 2 * p.W; hw += blockDim.x) {
        n += __popc(__ldcg(acc32 + hw));
        mp = max(mp, __ldcg(p.cp_pw + hw));
    }
    for (int o = 16; o; o >>= 1) {
        n += __shfl_xor_sync(0xFFFFFFFFu, n, o);
        mp = max(mp, __shfl_xor_sync(0xFFFFFFFFu, mp, o));
    }
    if (lane == 0) {
        if (n) atomicAdd(&s_n, (unsigned long long)n);
        atomicMax(&s_mp, mp);
    }
    __syncthreads();
    if (tid == 0) {
        *p.n_accepted = (long long)s_n;
        *p.passes_out = s_mp;
        *p.status_out = 0;
        if (p.status_user) *p.status_user = 0;
        *p.cp_done = 0;
        if (p.dbg) p.dbg[4] = globaltimer();
    }
}

cudaError_t launch_st_compact(const STParams &p, int blocks, size_t smem, cudaStream_t st, int threads) {
    st_compact_kernel<<<blocks, threads > 0 ? threads : kThreads, smem, st>>>(p);
    return cudaGetLastError();
}

// The compact matrix C[hw][A*] (uint32 columns) scattered into the (zeroed) matrix
// T0[n_ext][Wp] that lp_stable_matrix / lp_guess_model read (a thread per (atom, half-word),
// half-words fastest), and the all-ones rows (⊤, the facts) written over the valid guesses.
__global__ void st_expand_kernel(const uint32_t *C, const int32_t *atom, int32_t na, int32_t W, int64_t G,
                                 int32_t Wp, unsigned long long *T0, const int32_t *facts, int32_t nfacts,
                                 int32_t top) {
    const int64_t H = 2 * (int64_t)W;
    const int64_t total = (int64_t)na * H;
    uint32_t *T32 = reinterpret_cast<uint32_t *>(T0);
    const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, gn = (int64_t)gridDim.x * blockDim.x;
    for (int64_t x = gt; x < total; x += gn) {
        const int64_t a = x / H, hw = x % H;
        T32[(int64_t)__ldg(atom + a) * 2 * Wp + hw] = C[hw * na + a];
    }
    for (int64_t x = gt; x < (int64_t)(nfacts + 1) * W; x += gn) {
        const int64_t r = x / W, w = x % W;
        T0[(int64_t)(r == 0 ? top : __ldg(facts + r - 1)) * Wp + w] = valid_word(w, W, G);
    }
}

cudaError_t launch_st_expand(const STParams &p, cudaStream_t st) {
    const int64_t total = std::max<int64_t>((int64_t)p.cp_na * 2 * p.W, (int64_t)(p.nfacts + 1) * p.W);
    if (total == 0) return cudaSuccess;
    const int b = (int)std::min<int64_t>((total + 255) / 256, 8192);
    st_expand_kernel<<<b, 256, 0, st>>>(reinterpret_cast<const uint32_t *>(p.cp_C), p.cp_atom, p.cp_na, p.W, p.G,
                                        p.Wp, p.T0, p.facts, p.nfacts, p.top);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------
// guess-space reduction: sampling + local search (reading R23)
// ------------------------------------------------------------------------------------
//
// h columns per round: round 0 samples abar_j = rbit(seed, 0, g, j) for every free
// negated atom; a round runs the whole stable call above (clear, T_0 from the columns,
// Algorithm 2's loop, Algorithm 3's test); with no accepted column every column g flips
// the violated pairs j (a_j ∈ LM_g  ==  abar_j) whose rbit(seed, r+1, g, j) is 1, or one
// violated pair chosen by rand64(seed, r+1, g, k) if none is; then the next round -- all
// rounds in ONE cooperative launch.  Counter-based SplitMix64 (Steele, Lea, Flood 2014):
// rand64(seed, r, g, j) = mix(mix(mix(mix(seed) ^ r) ^ g) ^ j), rbit = rand64 >> 63.

__device__ __forceinline__ unsigned long long sm64_mix(unsigned long long z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// round 0: the columns of the initial matrix (a warp per (row j, 32 columns))
__device__ void search_sample(const STParams &p, int64_t gtid, int64_t gthreads) {
    const int lane = threadIdx.x & 31;
    const int64_t hw_n = 2 * (int64_t)p.W;                     // 32-column groups
    uint32_t *g32 = reinterpret_cast<uint32_t *>(p.gbuf);     // row j: 2W words
    const unsigned long long m1 = sm64_mix(sm64_mix(p.seed) ^ 0ull);
    for (int64_t t = gtid >> 5; t < (int64_t)p.k * hw_n; t += gthreads >> 5) {
        const int32_t j = (int32_t)(t / hw_n);
        const int64_t hw = t % hw_n;
        const int64_t g = hw * 32 + lane;
        bool b = false;
        if (g < p.G && p.free_rank[j] >= 0)
            b = (sm64_mix(sm64_mix(m1 ^ (unsigned long long)g) ^ (unsigned long long)j) >> 63) != 0;
        const unsigned w = __ballot_sync(0xFFFFFFFFu, b);
        if (lane == 0) g32[(int64_t)j * hw_n + hw] = w;
    }
}

// the local-search move from the fixpoint columns of round r_next - 1 (a warp per 32
// columns; T0 holds the fixpoint, gbuf the round's columns)
__device__ void search_move(const STParams &p, int32_t r_next, int64_t gtid, int64_t gthreads) {
    const int lane = threadIdx.x & 31;
    const int64_t hw_n = 2 * (int64_t)p.W;
    uint32_t *g32 = reinterpret_cast<uint32_t *>(p.gbuf);
    const uint32_t *T32 = reinterpret_cast<const uint32_t *>(p.T0);   // row a: 2Wp words
    const unsigned long long m2 = sm64_mix(sm64_mix(p.seed) ^ (unsigned long long)r_next);
    for (int64_t hw = gtid >> 5; hw < hw_n; hw += gthreads >> 5) {
        const int64_t g = hw * 32 + lane;
        const bool valid = g < p.G;
        const unsigned long long m3 = sm64_mix(m2 ^ (unsigned long long)g);
        int32_t nviol = 0, nflip = 0;
        for (int32_t j = 0; j < p.k; ++j) {
            const uint32_t bar = (__ldcg(g32 + (int64_t)j * hw_n + hw) >> lane) & 1u;
            const uint32_t inlm = (__ldcg(T32 + (int64_t)p.negated[j] * 2 * p.Wp + hw) >> lane) & 1u;
            const bool viol = bar + inlm != 1u;
            nviol += viol;
            nflip += viol && (sm64_mix(m3 ^ (unsigned long long)j) >> 63);
        }
        // no flip drawn: the violated pair number rand64(seed, r_next, g, k) mod |V_g|
        const int32_t sel = (nflip == 0 && nviol > 0)
                                ? (int32_t)(sm64_mix(m3 ^ (unsigned long long)p.k) % (unsigned long long)nviol)
                                : -1;
        int32_t cnt = 0;
        for (int32_t j = 0; j < p.k; ++j) {
            uint32_t *wp = g32 + (int64_t)j * hw_n + hw;
            const uint32_t bar = (__ldcg(wp) >> lane) & 1u;
            const uint32_t inlm = (__ldcg(T32 + (int64_t)p.negated[j] * 2 * p.Wp + hw) >> lane) & 1u;
            const bool viol = bar + inlm != 1u;
            bool flip;
            if (sel >= 0) {
                flip = viol && cnt == sel;
                cnt += viol;
            } else {
                flip = viol && (sm64_mix(m3 ^ (unsigned long long)j) >> 63);
            }
            const unsigned w = __ballot_sync(0xFFFFFFFFu, valid && ((bar ^ (flip ? 1u : 0u)) != 0u));
            if (lane == 0) *wp = w;
        }
    }
}

template <bool CL>
__global__ void __launch_bounds__(kThreads, 1) st_search_kernel(const __grid_constant__ STParams p) {
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gthreads = (int64_t)gridDim.x * blockDim.x;
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    __shared__ long long s_nacc;
    search_sample(p, gtid, gthreads);
    pass_barrier<CL>();
    int32_t passes = 0;
    for (int32_t r = 0;; ++r) {
        st_run<CL>(p, r == 0 ? p.clear_rows : 1);
        pass_barrier<CL>();   // (the check phase's accepted words and count are complete)
        if (threadIdx.x == 0) s_nacc = __ldcg(reinterpret_cast<const long long *>(p.n_accepted));
        __syncthreads();
        const long long nacc = s_nacc;
        if (lead) passes += *(volatile int32_t *)p.passes_out;
        if (nacc > 0 || r + 1 >= p.max_rounds) {
            if (lead) {
                *p.rounds_out = r + 1;
                *p.passes_sum_out = passes;
                if (p.status_user) *p.status_user = *(volatile int32_t *)p.status_out;
            }
            return;
        }
        search_move(p, r + 1, gtid, gthreads);
        pass_barrier<CL>();
    }
}

cudaError_t launch_st_search(const STParams &p, int blocks, size_t smem, cudaStream_t st, int cluster) {
    STParams q = p;
    return launch_grid_or_cluster(st_search_kernel<false>, st_search_kernel<true>, &q, sizeof(q), blocks, cluster,
                                  smem, st);
}

// The same search on the compact kernel's terms: CTA w
// owns guess word w in every round -- it samples its 64 columns, runs their fixpoint in
// shared memory, tests them and, from the fixpoint column still in shared memory, writes the
// NEXT round's columns (the local-search move) into the other column buffer; one grid
// barrier per round decides whether some column was accepted.  Same counter-based draws, so
// the same columns, rounds, passes and accepted ids as st_search_kernel and the oracle.
__global__ void __launch_bounds__(kThreads, 1) st_search_compact_kernel(const __grid_constant__ STParams p) {
    extern __shared__ __align__(16) unsigned long long cpb[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __shared__ int32_t s_cnt[4], s_rp;
    __shared__ long long s_nacc;
    cg::grid_group grid = cg::this_grid();
    const CpView v = cp_view(p, cpb, s_cnt);
    const int32_t na = v.na;
    const bool lead = blockIdx.x == 0 && tid == 0;
    const int32_t hw_n = 2 * p.W;
    unsigned long long *gb[2] = {p.gbuf, p.gbuf + (int64_t)p.k * p.W};
    uint32_t *C32 = reinterpret_cast<uint32_t *>(p.cp_C);
    uint32_t *acc32 = reinterpret_cast<uint32_t *>(p.accepted);
    int32_t cneg = -1, cabar = -1;
    if (tid < 32 && lane < p.k) {
        cneg = __ldg(p.cp_neg + lane);
        cabar = __ldg(p.cp_abar + lane);
    }
    if (lead) {
        *p.n_accepted = 0;
        p.cp_rp[0] = p.cp_rp[1] = p.cp_rp[2] = 0;
        *p.status_out = 0;
    }
    cp_stage(p, v);
    {   // round 0: the sampled columns of this CTA's half-words (a warp per row j)
        uint32_t *g32 = reinterpret_cast<uint32_t *>(gb[0]);
        const unsigned long long m1 = sm64_mix(sm64_mix(p.seed) ^ 0ull);
        for (int32_t hw = blockIdx.x; hw < hw_n; hw += gridDim.x)
            for (int32_t j = warp; j < p.k; j += (int32_t)(blockDim.x >> 5)) {
                const int64_t g = (int64_t)hw * 32 + lane;
                bool b = false;
                if (g < p.G && p.free_rank[j] >= 0)
                    b = (sm64_mix(sm64_mix(m1 ^ (unsigned long long)g) ^ (unsigned long long)j) >> 63) != 0;
                const unsigned wd = __ballot_sync(0xFFFFFFFFu, b);
                if (lane == 0) g32[(int64_t)j * hw_n + hw] = wd;
            }
    }
    grid.sync();   // (the counters are zero before any CTA adds to them)
    int32_t passes_sum = 0;
    for (int32_t r = 0;; ++r) {
        const unsigned long long *cols = gb[r & 1];
        uint32_t *nx32 = reinterpret_cast<uint32_t *>(gb[(r + 1) & 1]);
        const uint32_t *c32 = reinterpret_cast<const uint32_t *>(cols);
        if (lead) p.cp_rp[(r + 1) % 3] = 0;   // (last read two barriers ago)
        const unsigned long long m2 = sm64_mix(sm64_mix(p.seed) ^ (unsigned long long)(r + 1));
        for (int32_t hw = blockIdx.x; hw < hw_n; hw += gridDim.x) {
            const int32_t passes = cp_word<true>(p, v, hw, cols, false);
            for (int32_t a = tid; a < na; a += blockDim.x) C32[(int64_t)hw * na + a] = v.cur[a];
            if (tid < 32) {
                const uint32_t ok = cp_check(p, v, hw, cneg, cabar);
                if (lane == 0) {
                    acc32[hw] = ok;
                    if (ok) atomicAdd((unsigned long long *)p.n_accepted, (unsigned long long)__popc(ok));
                    atomicMax(p.cp_rp + r % 3, passes);
                }
            }
            // the local-search move of the half-word's columns (used only if no column of
            // the round is accepted): warp 1, a_j ∈ LM_g read from the fixpoint column in
            // shared memory
            if (warp == 1) {
                const int64_t g = (int64_t)hw * 32 + lane;
                const bool valid = g < p.G;
                const uint32_t vh = valid_half(p, hw);
                const unsigned long long m3 = sm64_mix(m2 ^ (unsigned long long)g);
                int32_t nviol = 0, nflip = 0;
                for (int32_t j = 0; j < p.k; ++j) {
                    const uint32_t bar = (__ldcg(c32 + (int64_t)j * hw_n + hw) >> lane) & 1u;
                    const uint32_t inlm = (cp_bits(v, __ldg(p.cp_neg + j), vh) >> lane) & 1u;
                    const bool viol = bar + inlm != 1u;
                    nviol += viol;
                    nflip += viol && (sm64_mix(m3 ^ (unsigned long long)j) >> 63);
                }
                const int32_t sel = (nflip == 0 && nviol > 0)
                                        ? (int32_t)(sm64_mix(m3 ^ (unsigned long long)p.k) % (unsigned long long)nviol)
                                        : -1;
                int32_t cnt = 0;
                for (int32_t j = 0; j < p.k; ++j) {
                    const uint32_t bar = (__ldcg(c32 + (int64_t)j * hw_n + hw) >> lane) & 1u;
                    const uint32_t inlm = (cp_bits(v, __ldg(p.cp_neg + j), vh) >> lane) & 1u;
                    const bool viol = bar + inlm != 1u;
                    bool flip;
                    if (sel >= 0) {
                        flip = viol && cnt == sel;
                        cnt += viol;
                    } else {
                        flip = viol && (sm64_mix(m3 ^ (unsigned long long)j) >> 63);
                    }
                    const unsigned wd = __ballot_sync(0xFFFFFFFFu, valid && ((bar ^ (flip ? 1u : 0u)) != 0u));
                    if (lane == 0) nx32[(int64_t)j * hw_n + hw] = wd;
                }
            }
            if (tid == 0) s_cnt[0] = s_cnt[1] = s_cnt[2] = s_cnt[3] = 0;
            __syncthreads();
        }
        grid.sync();
        if (tid == 0) {
            s_nacc = __ldcg(reinterpret_cast<const long long *>(p.n_accepted));
            s_rp = __ldcg(p.cp_rp + r % 3);
        }
        __syncthreads();
        const long long nacc = s_nacc;
        passes_sum += s_rp;
        if (nacc > 0 || r + 1 >= p.max_rounds) {
            if (r & 1) {   // the round's columns into the buffer the host reads
                const uint32_t *src = reinterpret_cast<const uint32_t *>(gb[1]);
                uint32_t *dst = reinterpret_cast<uint32_t *>(gb[0]);
                for (int32_t hw = blockIdx.x; hw < hw_n; hw += gridDim.x)
                    for (int32_t j = tid; j < p.k; j += blockDim.x)
                        dst[(int64_t)j * hw_n + hw] = __ldcg(src + (int64_t)j * hw_n + hw);
            }
            if (lead) {
                *p.rounds_out = r + 1;
                *p.passes_sum_out = passes_sum;
                *p.passes_out = s_rp;
                if (p.status_user) *p.status_user = 0;
            }
            return;
        }
        __syncthreads();   // (s_nacc / s_rp are rewritten after the next barrier)
    }
}

// co-resident CTAs per SM of the compact kernels with `smem` bytes (which: 0 stable, 1 search)
int st_compact_blocks_per_sm(int which, size_t smem) {
    int a = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &a, which ? (const void *)st_search_compact_kernel : (const void *)st_compact_kernel, kThreads, smem);
    return a;
}

cudaError_t launch_st_search_compact(const STParams &p, int blocks, size_t smem, cudaStream_t st) {
    STParams q = p;
    void *args[] = {(void *)&q};
    return cudaLaunchCooperativeKernel((const void *)st_search_compact_kernel, dim3(blocks), dim3(kThreads), args,
                                       smem, st);
}

cudaError_t launch_st_fused(const STParams &p, int blocks, size_t smem, cudaStream_t st, int cluster) {
    STParams q = p;
    return launch_grid_or_cluster(st_fixpoint_kernel<false>, st_fixpoint_kernel<true>, &q, sizeof(q), blocks,
                                  cluster, smem, st);
}

// Algorithm 3 (reading R7): guess g is accepted iff for every negated
// atom a_j, T[a_j] + T[abar_j] = 1 in column g, i.e. the XOR of the two rows is 1.
__global__ void st_column_kernel(const unsigned long long *T, int32_t Wp, int32_t n, int64_t g,
                                 unsigned long long *out) {
    const int64_t nw = ((int64_t)n + 63) >> 6;
    const int64_t gw = g >> 6;
    const int gb = (int)(g & 63);
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nw;
         w += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long v = 0;
        for (int b = 0; b < 64; ++b) {
            const int64_t a = w * 64 + b;
            if (a >= n) break;
            v |= ((T[a * Wp + gw] >> gb) & 1ull) << b;
        }
        out[w] = v;
    }
}

cudaError_t launch_st_column(const STParams &p, int32_t n, int64_t g, unsigned long long *out,
                             cudaStream_t st) {
    const int64_t nw = ((int64_t)n + 63) >> 6;
    if (nw == 0) return cudaSuccess;
    int b = (int)std::min<int64_t>((nw + 255) / 256, 4096);
    st_column_kernel<<<b, 256, 0, st>>>(p.T0, p.Wp, n, g, out);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------
// multi-GPU least model: the exchange step of a head-range-sharded pass
// ------------------------------------------------------------------------------------
//
// After every rank ran ONE θ-pass of its rules (heads in its 64-aligned atom range) from
// the same v_k and the ranks' owned words were all-gathered: v_{k+1} = v_k with each
// rank's owned words ORed in (the OR clause of T_P over rules split across GPUs), the
// changed flag = some rank's pass derived an atom (its status word has LP_ST_CAPPED), and
// optionally |v_{k+1}| added to *pops.  Block 0 writes the flag (a plain store: the host
// may read it from mapped memory once the stream passed the kernel).
__global__ void shard_combine_kernel(const __grid_constant__ ShardCombineParams q) {
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gthreads = (int64_t)gridDim.x * blockDim.x;
    int32_t pc = 0;
    for (int64_t w = gtid; w < q.n_words; w += gthreads) {
        int r = 0;
        while (r + 1 < q.world && q.word_lo[r + 1] <= w) ++r;   // (ranges ascending, <= 64)
        unsigned long long v = __ldg(q.v + w);
        const int64_t i = w - q.word_lo[r];
        if (i < q.word_cnt[r]) v |= __ldg(q.gathered + (int64_t)r * q.stride + i);
        q.v_next[w] = v;
        pc += __popcll(v);
    }
    if (q.pops) {
        for (int o = 16; o; o >>= 1) pc += __shfl_xor_sync(0xFFFFFFFFu, pc, o);
        if ((threadIdx.x & 31) == 0 && pc) atomicAdd(q.pops, pc);
    }
    if (blockIdx.x == 0 && threadIdx.x < 32) {
        int32_t ch = 0;
        for (int r = threadIdx.x; r < q.world; r += 32) {
            const int32_t st = (int32_t)__ldg(q.gathered + (int64_t)r * q.stride + (q.stride - 1));
            ch |= (st & kStCapped) ? 1 : 0;
        }
        ch = __any_sync(0xFFFFFFFFu, ch != 0) ? 1 : 0;
        if (threadIdx.x == 0) *(volatile int32_t *)q.changed = ch;
    }
}

cudaError_t launch_shard_combine(const ShardCombineParams &q, cudaStream_t st) {
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((q.n_words + 255) / 256, 4 * 148));
    shard_combine_kernel<<<(unsigned)blocks, 256, 0, st>>>(q);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------
// occupancy
// ------------------------------------------------------------------------------------

cudaError_t prepare_kernels(size_t lm_smem, size_t st_smem) {
    cudaError_t e;
    const int cap = std::max(kMaxSmemBytes, kKeySmemBytes);   // + static smem <= 227 KB
    (void)lm_smem;
    (void)st_smem;
    const void *full[4] = {(const void *)lm_full_kernel<true, false>, (const void *)lm_full_kernel<false, false>,
                           (const void *)lm_full_kernel<true, true>, (const void *)lm_full_kernel<false, true>};
    for (const void *k : full)
        if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, cap))) return e;
    if ((e = cudaFuncSetAttribute((const void *)st_fixpoint_kernel<false>,   // (+ its static candidate queue)
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmemBytes)))
        return e;
    if ((e = cudaFuncSetAttribute((const void *)st_search_kernel<false>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmemBytes)))
        return e;
    if ((e = cudaFuncSetAttribute((const void *)lm_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kMaxSmemBytes)))
        return e;
    if ((e = cudaFuncSetAttribute((const void *)st_compact_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kCpSmemBytes)))
        return e;
    if ((e = cudaFuncSetAttribute((const void *)st_search_compact_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kCpSmemBytes)))
        return e;
    // the one-cluster launches of the same kernels (16 CTAs: a non-portable cluster size)
    const void *cl[3] = {(const void *)st_fixpoint_kernel<true>, (const void *)st_search_kernel<true>,
                         (const void *)lm_frontier_kernel<true>};
    for (const void *k : cl) {
        if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmemBytes))) return e;
        if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1))) return e;
    }
    return cudaSuccess;
}

int lm_full_blocks_per_sm(bool exact, size_t smem) {
    int nb = 0, na = 0;   // (both instantiations run on the same grid)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &nb, exact ? (const void *)lm_full_kernel<true, false> : (const void *)lm_full_kernel<false, false>,
        kFullThreads, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &na, exact ? (const void *)lm_full_kernel<true, true> : (const void *)lm_full_kernel<false, true>,
        kFullThreads, smem);
    return std::min(nb, na);
}

int lm_frontier_blocks_per_sm() {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void *)lm_frontier_kernel<false>, kThreads, 0);
    return nb;
}

int st_blocks_per_sm(size_t smem) {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void *)st_fixpoint_kernel<false>, kThreads, smem);
    int ns = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ns, (const void *)st_search_kernel<false>, kThreads, smem);
    return std::min(nb, ns);   // (both launch on the same grid)
}

}  // namespace lpb

namespace lpb {
// The largest one-cluster launch (<= want CTAs) of the cluster instantiation of a
// persistent kernel with `smem` bytes: 0 if none fits.  which: 0 frontier, 1 stable.
int cluster_size_for(int which, int want, size_t smem) {
    const void *ks[2][2] = {{(const void *)lm_frontier_kernel<true>, nullptr},
                            {(const void *)st_fixpoint_kernel<true>, (const void *)st_search_kernel<true>}};
    for (int c = want; c >= 1; --c) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)c);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)c;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        bool ok = true;
        for (const void *k : ks[which]) {
            int n = 0;
            if (!k) continue;
            if (cudaOccupancyMaxActiveClusters(&n, k, &cfg) != cudaSuccess || n < 1) ok = false;
        }
        cudaGetLastError();
        if (ok) return c;
    }
    return 0;
}
}  // namespace lpb
