// C ABI (include/lp.h): device residency, launch configuration and the three calls of
// the boundary: lp_load, lp_least_model, lp_stable_models.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "kernels.h"

using namespace lpb;

static thread_local std::string g_err;

static lp_status set_err(lp_status s, const std::string &m) {
    g_err = m;
    return s;
}

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess)                                                             \
            return set_err(LP_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));    \
    } while (0)

struct lp_program {
    HostLayout L;
    int device = -1;
    lp_alloc_fn af = nullptr;
    lp_free_fn ff = nullptr;
    void *actx = nullptr;
    std::vector<std::pair<void *, size_t>> allocs;
    int64_t dev_bytes = 0;
    int guess_cap = 20;

    Segment *d_segs = nullptr;
    int32_t *d_col = nullptr, *d_head = nullptr;
    int64_t *d_occ_ptr = nullptr;
    int32_t *d_occ_slot = nullptr;
    int32_t *d_fq = nullptr;   // frontier level queues [2][n_ext + 1] x (atom, occ range, -)
    uint32_t *d_cnt = nullptr;
    int cnt_bits = 8;
    uint32_t *d_buf0 = nullptr, *d_buf1 = nullptr;
    int32_t nwords = 0;
    uint32_t *d_summary = nullptr;
    int32_t sm_words = 0, shift = 0;
    bool exact = true;
    int32_t *d_order = nullptr;
    int32_t *d_qbuf = nullptr;  // FILTER-mode candidate queues, [lm_blocks][qcap]
    int32_t qcap = 0;
    // A/B switches of the measurements (environment, read once by lp_load; every setting
    // computes the same results -- DESIGN.md "A/B switches")
    int32_t dense_div = 16;     // LP_DENSE_DIV: auto schedule's queued-rows divisor
    bool env_no_pipe = false;   // LP_NO_PIPE
    bool env_no_predict = false;  // LP_NO_PREDICT
    bool env_no_overlap = false;  // LP_NO_OVERLAP
    bool env_no_ksum_image = false;  // LP_NO_KSUM_IMAGE
    bool env_no_zerocopy = false;    // LP_NO_ZEROCOPY
    bool env_no_prefetch = false;    // LP_NO_PREFETCH
    long long overlap_min_bytes = 16ll << 20;   // LP_OVERLAP_MIN_MB: overlapped / pipelined
                                                // LEAD passes from this live stream size on
    // [0] tail, [2] status (stable path); [1] iters; [3] passes; [4,5] n_accepted;
    // [6] search rounds, [7] search passes (sum over rounds);
    // [8,9] least-model tails and [10,11] statuses, alternating by call parity;
    // [12..14] rows queued per full θ-pass (slot k % 3); [16..18] least-model and
    // [20..22] stable per-pass append counters (slot k % 3); [26] compact stable kernel:
    // CTAs finished (self-resetting)
    int32_t *d_scal = nullptr;
    // host-pointer calls: iters and the status word written by the kernel's epilogue into
    // page-locked mapped memory (no scalar copies after the launch); NULL if unavailable
    int32_t *h_scal = nullptr, *h_scal_dev = nullptr;
    unsigned long long *d_stats = nullptr;  // full θ-pass work statistics (lp_run.stats_out)
    unsigned long long *d_vent = nullptr;   // [3] entries verified per pass (schedule)
    int32_t *d_cand = nullptr;   // [3] rows queued per full θ-pass (slot k % 3), on a line of
                                 // its own: the pass's append counters (d_scal) are the line
                                 // every CTA reads right after each barrier
    void *d_lead_codes = nullptr;   // summary-mode key plane (low key_bits bits of the lead group)
    void *d_octet_tag = nullptr;    // per-octet bucket | padding tags
    int key_bits = 16;
    int32_t *d_lead32 = nullptr;    // exact mode: flat lead plane
    uint16_t *d_xlead16 = nullptr, *d_xhead16 = nullptr, *d_xtag = nullptr;   // exact 16-bit planes
    int32_t *d_key_of = nullptr;
    int4 *d_runs = nullptr;         // key mode: bucket runs (first octet, octets, bucket, 0)
    int32_t nruns = 0;              //   0: no table (LEAD passes stream every octet)
    int32_t *d_korder = nullptr;
    int32_t ksm_words = 0, kshift = 0;
    uint32_t *d_factbits = nullptr, *d_init_bits = nullptr;
    int32_t *d_init_list = nullptr, *d_init_klist = nullptr;
    uint32_t *d_init_ksum = nullptr;
    int32_t *d_locc_ptr = nullptr, *d_locc_slot = nullptr;
    // exact mode, armed LEAD passes: rows by lead atom
    // (arm_ptr[a] .. arm_ptr[a+1]) as 32-byte records, and the per-CTA list capacity
    int32_t *d_arm_ptr = nullptr;
    int4 *d_arec = nullptr;
    int32_t arm_cap = 0;
    int64_t n_records = 0;
    int32_t st_arm_cap = 0;   // stable: records owned per CTA (0: the scan)
    int32_t n_init = 0;
    uint64_t lm_runs = 0;
    int32_t *d_facts = nullptr;
    int32_t nfacts = 0;
    int32_t *d_negated = nullptr, *d_negated_ext = nullptr, *d_free_rank = nullptr;
    unsigned long long *d_v0 = nullptr, *d_model = nullptr;
    int32_t *d_stage = nullptr, *d_pops = nullptr;
    int32_t pops_alloc = 0;

    unsigned long long *d_T0 = nullptr, *d_T1 = nullptr;
    size_t T_words_alloc = 0;
    int32_t W = 0, Wp = 0;
    int64_t G = 0;
    bool stable_valid = false;
    uint32_t *d_any = nullptr, *d_gfull = nullptr;
    int32_t any_words = 0, any_shift = 0;
    bool st_full = false;
    int32_t *d_mark = nullptr;
    int32_t *d_st_ring = nullptr;   // stable: per-pass lists (ring of 3)
    bool st_dirty_ok = false;   // T holds only the previous call's dirty rows (same Wp)
    int32_t st_last_Wp = 0;
    unsigned long long *d_acc = nullptr, *d_guess = nullptr;
    size_t acc_words_alloc = 0, guess_words_alloc = 0;
    unsigned long long *d_sguess = nullptr;   // lp_stable_search: the round's columns [k][W]
    size_t sguess_words_alloc = 0;
    // compact stable kernel: the live sub-program
    bool cp_ok = false;
    int32_t cp_na = 0, cp_nr = 0, cp_nnz = 0, cp_n0 = 0, cp_blob16 = 0;
    size_t cp_smem = 0;
    int cp_occ = 1, cp_occ_search = 1;   // co-resident CTAs per SM of the compact kernels
    int cp_threads = 0;                  // LP_CP_THREADS: threads per CTA of st_compact_kernel (0: kThreads)
    uint4 *d_cp_blob = nullptr;
    int32_t *d_cp_atom = nullptr, *d_cp_neg = nullptr, *d_cp_abar = nullptr;
    int32_t *d_cp_pw = nullptr, *d_cp_rp = nullptr;
    size_t cp_pw_alloc = 0;
    unsigned long long *d_cp_C = nullptr;   // [W][na] the last compact call's fixpoint matrix over A*
    size_t cp_C_alloc = 0;
    bool st_last_compact = false;   // the last stable call ran the compact kernel (result in C) ...
    bool cp_expanded = false;       // ... and C was scattered into T0 for a readback

    int cluster = 0;            // > 0: exact-mode program run by ONE cluster of this many CTAs
    int cl_threads = 0;         // ... with this many threads per CTA (0: kThreads; LP_CLUSTER_THREADS)
    int fr_cl_threads = 0;      // one-cluster frontier launches: threads per CTA (LP_FR_CLUSTER_THREADS)
    size_t cluster_smem = 0;
    bool cluster_stage = false; // ... with the program planes staged in shared memory
    // small-program kernel: the rows in shared memory
    bool small_ok = false;
    uint4 *d_sm_blob = nullptr;
    int32_t sm_blob16 = 0, sm_nr = 0, sm_nnz = 0;
    size_t small_smem = 0;
    int small_threads = 0;   // LP_SMALL_THREADS: threads of lm_small_kernel's CTA (0: 512)
    int sms = 0, threads = kThreads;
    int lm_blocks = 0, fr_blocks = 0, st_blocks = 0, grid_cap = 0;
    int fr_cluster = 0, st_cluster = 0;   // > 0: one-cluster launch of the frontier / stable kernels
    size_t lm_smem = 0, st_smem = 0;
};

// ------------------------------------------------------------------------------------
// device memory
// ------------------------------------------------------------------------------------

static lp_status dev_alloc(lp_program *p, size_t bytes, void **out) {
    bytes = std::max<size_t>(bytes, 16);
    bytes = (bytes + 255) / 256 * 256;
    void *ptr = nullptr;
    if (p->af) {
        ptr = p->af(bytes, p->actx);
        if (!ptr) return set_err(LP_E_NOMEM, "device allocation hook failed");
    } else {
        cudaError_t e = cudaMalloc(&ptr, bytes);
        if (e != cudaSuccess)
            return set_err(LP_E_NOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    }
    p->allocs.emplace_back(ptr, bytes);
    p->dev_bytes += (int64_t)bytes;
    *out = ptr;
    return LP_OK;
}

template <class T>
static lp_status dalloc(lp_program *p, T **out, size_t count) {
    void *v = nullptr;
    lp_status s = dev_alloc(p, count * sizeof(T), &v);
    *out = (T *)v;
    return s;
}

static void dev_release(lp_program *p, void *ptr) {
    for (size_t i = 0; i < p->allocs.size(); ++i) {
        if (p->allocs[i].first != ptr) continue;
        if (p->ff) p->ff(ptr, p->allocs[i].second, p->actx);
        else cudaFree(ptr);
        p->dev_bytes -= (int64_t)p->allocs[i].second;
        p->allocs.erase(p->allocs.begin() + (long)i);
        return;
    }
}

template <class T>
static lp_status upload(lp_program *p, T **out, const std::vector<T> &v) {
    lp_status s = dalloc(p, out, std::max<size_t>(v.size(), 1));
    if (s) return s;
    if (!v.empty()) CK(cudaMemcpy(*out, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    return LP_OK;
}

#define TRY(x)                          \
    do {                                \
        lp_status s_ = (x);             \
        if (s_ != LP_OK) return s_;     \
    } while (0)

// Program bytes one full θ-pass streams: a LEAD pass reads
// the lead plane (+ the head plane when the truth test is exact), a STREAM pass every
// body plane (+ the head plane when exact).  Padding rows included.
static uint64_t lead_plane_bytes(const lp_program *p) {
    if (p->d_lead_codes)   // key plane + octet tags
        return p->key_bits == 8 ? (uint64_t)p->L.n_slots + (uint64_t)p->L.n_slots / 4
                                : 2ull * (uint64_t)p->L.n_slots + (uint64_t)p->L.n_slots / 8;
    if (p->d_xlead16) return 4ull * (uint64_t)p->L.n_slots + (uint64_t)p->L.n_slots / 4;  // 16-bit lead + head + tags
    uint64_t b = 4ull * (uint64_t)p->L.n_slots;
    return p->exact ? 2 * b : b;
}

static uint64_t stream_plane_bytes(const lp_program *p) {
    uint64_t b = 0;
    for (const Segment &sg : p->L.segs) b += 4ull * (uint64_t)sg.L * (uint64_t)sg.count_pad;
    return p->exact ? b + 4ull * (uint64_t)p->L.n_slots : b;
}

// ------------------------------------------------------------------------------------
// lp_load
// ------------------------------------------------------------------------------------

// LP_LOAD_TIMING=1: lp_load prints the host time of each phase to stderr (profiling aid)
static void load_mark(const char *what) {
    static thread_local std::chrono::steady_clock::time_point t0;
    static const bool on = std::getenv("LP_LOAD_TIMING") != nullptr;
    if (!on) return;
    const auto t = std::chrono::steady_clock::now();
    if (what) std::fprintf(stderr, "lp_load %-28s %8.3f s\n", what, std::chrono::duration<double>(t - t0).count());
    t0 = t;
}

// The live sub-program of a normal program for the compact stable kernel: A* = the least
// model of P+ (Eq. 4) from the facts, ⊤ and EVERY abar_j -- P+ is definite, so A* contains
// the least model of every guess (Def. 8 only takes abar_j away) -- by counter forward
// chaining over the encoded rows; a row can fire in some guess only if its body lies in A*.
// Kept (compact ids, ascending extended atom id; rows in slot order) when it fits the
// kernel's shared memory next to the two column buffers; rows whose head is a fact or ⊤
// (all ones from T_0 on) are dropped.
static lp_status build_compact_stable(lp_program *p) {
    const HostLayout &L = p->L;
    const int32_t ne = L.n_ext;
    std::vector<uint8_t> tr((size_t)ne, 0), ones((size_t)ne, 0);
    std::vector<int32_t> queue;
    auto set_true = [&](int32_t a) {
        if (!tr[a]) { tr[a] = 1; queue.push_back(a); }
    };
    set_true(L.top);
    ones[L.top] = 1;
    for (int32_t a : L.facts) { set_true(a); ones[a] = 1; }
    for (int32_t a : L.st_facts) { set_true(a); ones[a] = 1; }
    for (int32_t j = 0; j < L.k; ++j) set_true(L.n + j);
    // occurrence lists over the real slots (every body position)
    std::vector<int64_t> optr((size_t)ne + 1, 0);
    for (const Segment &sg : L.segs)
        for (int32_t j = 0; j < sg.L; ++j)
            for (int64_t i = 0; i < sg.count; ++i) ++optr[(size_t)L.col[sg.col_off + (int64_t)j * sg.count_pad + i] + 1];
    for (int32_t a = 0; a < ne; ++a) optr[a + 1] += optr[a];
    if (optr[ne] > INT32_MAX || L.n_slots > INT32_MAX) return LP_OK;   // (no compact kernel)
    std::vector<int32_t> oslot((size_t)optr[ne]), cnt((size_t)L.n_slots, 0);
    {
        std::vector<int64_t> fill(optr.begin(), optr.end() - 1);
        for (const Segment &sg : L.segs)
            for (int64_t i = 0; i < sg.count; ++i) {
                cnt[sg.slot_off + i] = sg.L;
                for (int32_t j = 0; j < sg.L; ++j)
                    oslot[(size_t)fill[L.col[sg.col_off + (int64_t)j * sg.count_pad + i]]++] = (int32_t)(sg.slot_off + i);
            }
    }
    std::vector<uint8_t> live((size_t)L.n_slots, 0);
    for (size_t qi = 0; qi < queue.size(); ++qi) {
        const int32_t a = queue[qi];
        for (int64_t o = optr[a]; o < optr[a + 1]; ++o) {
            const int32_t s = oslot[(size_t)o];
            if (--cnt[s] == 0) {
                live[s] = 1;
                set_true(L.head[s]);
            }
        }
    }
    // compact ids for A* minus the all-ones atoms (⊤, the facts: they never mask a bit and
    // never change; -2 stands for them where a compact id is expected)
    std::vector<int32_t> cid((size_t)ne, -1), atom, init;
    for (int32_t a = 0; a < ne; ++a)
        if (tr[a]) {
            if (ones[a]) {
                cid[a] = -2;
                continue;
            }
            cid[a] = (int32_t)atom.size();
            atom.push_back(a);
            init.push_back((a >= L.n && a < L.n + L.k) ? a - L.n : -1);
        }
    if (atom.size() > 65534 || L.k > 32767) return LP_OK;
    const size_t na = atom.size();
    std::vector<uint16_t> rptr(1, (uint16_t)0), rhead, rbody;
    for (const Segment &sg : L.segs)
        for (int64_t i = 0; i < sg.count; ++i) {
            const int64_t s = sg.slot_off + i;
            if (!live[s] || ones[L.head[s]]) continue;
            if (rhead.size() >= 65535 || rbody.size() + (size_t)sg.L > 65535) return LP_OK;
            rhead.push_back((uint16_t)cid[L.head[s]]);
            for (int32_t j = 0; j < sg.L; ++j) {
                const int32_t b = L.col[sg.col_off + (int64_t)j * sg.count_pad + i];
                if (!ones[b]) rbody.push_back((uint16_t)cid[b]);   // (all-ones rows never mask a bit)
            }
            rptr.push_back((uint16_t)rbody.size());
        }
    const size_t nr = rhead.size(), nz = rbody.size();
    // the transpose: the live rows in which compact atom c occurs
    std::vector<uint16_t> cptr(na + 1, 0), crow(nz);
    {
        std::vector<uint32_t> c32(na + 1, 0u);
        for (uint16_t b : rbody) ++c32[(size_t)b + 1];
        for (size_t c = 0; c < na; ++c) c32[c + 1] += c32[c];
        for (size_t c = 0; c <= na; ++c) cptr[c] = (uint16_t)c32[c];
        for (size_t r = 0; r < nr; ++r)
            for (uint32_t i = rptr[r]; i < rptr[r + 1]; ++i) crow[c32[rbody[i]]++] = (uint16_t)r;
    }
    // pass 0 can fire only rows whose remaining body atoms are abar atoms (T_0 is zero elsewhere)
    std::vector<uint16_t> row0;
    for (size_t r = 0; r < nr; ++r) {
        bool ok = true;
        for (uint32_t i = rptr[r]; i < rptr[r + 1] && ok; ++i) ok = init[rbody[i]] >= 0;
        if (ok) row0.push_back((uint16_t)r);
    }
    const size_t n0 = row0.size();
    const size_t blob_bytes = (2 * (4 * nr + nz + (na + 1) + nz + na + n0) + 15) / 16 * 16;
    const size_t smem = blob_bytes + 8 * na + 2 * (na + (na & 1)) + 4 * (nz + (nz & 1));
    if (smem > (size_t)kCpSmemBytes) return LP_OK;
    std::vector<uint4> blob(blob_bytes / 16, make_uint4(0, 0, 0, 0));
    {
        uint16_t *b = reinterpret_cast<uint16_t *>(blob.data());
        auto put = [&](const void *src, size_t n16) {
            if (n16) std::memcpy(b, src, 2 * n16);
            b += n16;
        };
        std::vector<uint16_t> rrec(4 * nr);
        for (size_t r = 0; r < nr; ++r) {
            rrec[4 * r] = rhead[r];
            rrec[4 * r + 1] = rptr[r];
            rrec[4 * r + 2] = rptr[r + 1];
            rrec[4 * r + 3] = rptr[r + 1] > rptr[r] ? rbody[rptr[r]] : (uint16_t)0xFFFF;   // (kCpNone)
        }
        put(rrec.data(), 4 * nr);
        put(rbody.data(), nz);
        put(cptr.data(), na + 1);
        put(crow.data(), nz);
        std::vector<int16_t> i16(init.begin(), init.end());
        put(i16.data(), na);
        put(row0.data(), n0);
    }
    std::vector<int32_t> cneg(L.k), cabar(L.k);
    for (int32_t j = 0; j < L.k; ++j) {
        cneg[j] = cid[L.negated[j]];
        cabar[j] = cid[L.n + j];
    }
    TRY(upload(p, &p->d_cp_blob, blob));
    TRY(upload(p, &p->d_cp_atom, atom));
    TRY(upload(p, &p->d_cp_neg, cneg));
    TRY(upload(p, &p->d_cp_abar, cabar));
    TRY(upload(p, &p->d_cp_rp, std::vector<int32_t>(4, 0)));
    p->cp_na = (int32_t)na;
    p->cp_nr = (int32_t)nr;
    p->cp_nnz = (int32_t)nz;
    p->cp_n0 = (int32_t)n0;
    p->cp_blob16 = (int32_t)(blob_bytes / 16);
    p->cp_smem = smem;
    p->cp_ok = true;
    return LP_OK;
}

// The rows of a small program for lm_small_kernel: 16-bit extended atom ids, rows in slot
// order; a row whose head is a fact is dropped (v_0 holds its head), and so are the body
// atoms that are facts or ⊤ (true in every v_k).
static lp_status build_small(lp_program *p) {
    const HostLayout &L = p->L;
    const size_t ne = (size_t)L.n_ext;
    if (ne > 65534 || L.n_slots > 65535) return LP_OK;
    std::vector<uint8_t> ones(ne, 0);
    ones[L.top] = 1;
    for (int32_t a : L.facts) ones[a] = 1;
    std::vector<uint16_t> rptr(1, (uint16_t)0), rhead, rbody;
    for (const Segment &sg : L.segs)
        for (int64_t i = 0; i < sg.count; ++i) {
            const int32_t h = L.head[sg.slot_off + i];
            if (ones[h]) continue;
            if (rbody.size() + (size_t)sg.L > 65535) return LP_OK;
            rhead.push_back((uint16_t)h);
            for (int32_t j = 0; j < sg.L; ++j) {
                const int32_t b = L.col[sg.col_off + (int64_t)j * sg.count_pad + i];
                if (!ones[b]) rbody.push_back((uint16_t)b);
            }
            rptr.push_back((uint16_t)rbody.size());
        }
    const size_t nr = rhead.size(), nz = rbody.size();
    std::vector<uint16_t> cptr(ne + 1, 0), crow(nz);
    {
        std::vector<uint32_t> c32(ne + 1, 0u);
        for (uint16_t b : rbody) ++c32[(size_t)b + 1];
        for (size_t c = 0; c < ne; ++c) c32[c + 1] += c32[c];
        for (size_t c = 0; c <= ne; ++c) cptr[c] = (uint16_t)c32[c];
        for (size_t r = 0; r < nr; ++r)
            for (uint32_t i = rptr[r]; i < rptr[r + 1]; ++i) crow[c32[rbody[i]]++] = (uint16_t)r;
    }
    const size_t blob_bytes = (2 * (4 * nr + nz + (ne + 1) + nz) + 15) / 16 * 16;
    const size_t smem = blob_bytes + 8 * (size_t)p->nwords + 2 * (ne + (ne & 1)) + 4 * (nz + (nz & 1));
    if (smem > (size_t)kMaxSmemBytes) return LP_OK;
    std::vector<uint4> blob(blob_bytes / 16, make_uint4(0, 0, 0, 0));
    {
        uint16_t *b = reinterpret_cast<uint16_t *>(blob.data());
        auto put = [&](const void *src, size_t n16) {
            if (n16) std::memcpy(b, src, 2 * n16);
            b += n16;
        };
        std::vector<uint16_t> rrec(4 * nr);
        for (size_t r = 0; r < nr; ++r) {
            rrec[4 * r] = rhead[r];
            rrec[4 * r + 1] = rptr[r];
            rrec[4 * r + 2] = rptr[r + 1];
            rrec[4 * r + 3] = rptr[r + 1] > rptr[r] ? rbody[rptr[r]] : (uint16_t)0xFFFF;
        }
        put(rrec.data(), 4 * nr);
        put(rbody.data(), nz);
        put(cptr.data(), ne + 1);
        put(crow.data(), nz);
    }
    TRY(upload(p, &p->d_sm_blob, blob));
    p->sm_blob16 = (int32_t)(blob_bytes / 16);
    p->sm_nr = (int32_t)nr;
    p->sm_nnz = (int32_t)nz;
    p->small_smem = smem;
    p->small_ok = true;
    return LP_OK;
}

static lp_status load_device(lp_program *p, const lp_options *opt) {
    HostLayout &L = p->L;
    load_mark(nullptr);
    CK(cudaSetDevice(p->device));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device));
    p->sms = sms;

    {   // rows of the stable initial matrix set to 1 (Def. 8 item 2)
        std::vector<int32_t> sf(L.facts);
        sf.insert(sf.end(), L.st_facts.begin(), L.st_facts.end());
        TRY(upload(p, &p->d_facts, sf));
        p->nfacts = (int32_t)sf.size();
    }
    TRY(upload(p, &p->d_negated, L.negated));
    {
        std::vector<int32_t> ext(L.k), rank(L.k, -1);
        for (int32_t j = 0; j < L.k; ++j) ext[j] = L.n + j;
        for (size_t i = 0; i < L.free_j.size(); ++i) rank[L.free_j[i]] = (int32_t)i;
        TRY(upload(p, &p->d_negated_ext, ext));
        TRY(upload(p, &p->d_free_rank, rank));
    }
    // truth vector: bit a of word a>>5, padded to a multiple of 4 words (int4 loads)
    p->nwords = (int32_t)((((int64_t)L.n_ext + 31) / 32 + 3) / 4 * 4);
    TRY(dalloc(p, &p->d_buf0, p->nwords));
    TRY(dalloc(p, &p->d_buf1, p->nwords));
    TRY(dalloc(p, &p->d_order, (size_t)L.n_ext + 1));
    TRY(dalloc(p, &p->d_scal, 32));
    {   // (best effort: without it host-pointer calls copy the scalars back)
        void *h = nullptr;
        if (cudaHostAlloc(&h, 64, cudaHostAllocMapped) == cudaSuccess) {
            void *hd = nullptr;
            if (cudaHostGetDevicePointer(&hd, h, 0) == cudaSuccess) {
                p->h_scal = static_cast<int32_t *>(h);
                p->h_scal_dev = static_cast<int32_t *>(hd);
            } else {
                cudaFreeHost(h);
            }
        }
        cudaGetLastError();
    }
    CK(cudaMemset(p->d_scal, 0, 32 * sizeof(int32_t)));
    TRY(dalloc(p, &p->d_stats, 6));
    TRY(dalloc(p, &p->d_vent, 3));
    TRY(dalloc(p, &p->d_cand, 32));
    CK(cudaMemset(p->d_cand, 0, 32 * sizeof(int32_t)));
    {
        std::vector<uint32_t> fb((size_t)p->nwords, 0u);   // facts of P (Def. 4)
        for (int32_t a : L.facts) fb[(size_t)a >> 5] |= 1u << (a & 31);
        TRY(upload(p, &p->d_factbits, fb));
        fb[(size_t)L.top >> 5] |= 1u << (L.top & 31);        // v_0 for v0 == NULL: + ⊤
        TRY(upload(p, &p->d_init_bits, fb));
        TRY(upload(p, &p->d_init_list, L.facts));           // its derivation list (ids ascending)
        p->n_init = (int32_t)L.facts.size();
    }
    const size_t mw = std::max<size_t>(((size_t)L.n_out + 63) / 64, 1);
    TRY(dalloc(p, &p->d_v0, mw));
    TRY(dalloc(p, &p->d_model, mw));

    // shared-memory plan: exact truth vector if it fits, else a summary
    int64_t cap = kMaxSmemBytes;
    if (opt && opt->smem_bits_cap > 0) cap = std::min<int64_t>(cap, opt->smem_bits_cap / 8);
    cap = std::max<int64_t>(cap, 16);
    if ((int64_t)p->nwords * 4 <= cap) {
        p->exact = true;
        p->shift = 0;
        p->sm_words = p->nwords;
    } else {
        p->exact = false;
        int sh = 1;
        for (;; ++sh) {
            const int64_t groups = (((int64_t)L.n_ext - 1) >> sh) + 1;
            const int64_t w = ((groups + 31) / 32 + 3) / 4 * 4;
            if (w * 4 <= cap) { p->sm_words = (int32_t)w; break; }
        }
        p->shift = sh;
        TRY(dalloc(p, &p->d_summary, p->sm_words));
        CK(cudaMemset(p->d_summary, 0, (size_t)p->sm_words * 4));   // zero between calls
    }
    p->lm_smem = (size_t)p->sm_words * 4;

    load_mark("small uploads");
    // key plane (summary mode, register-streaming kernel): every
    // extended atom gets a key -- atoms that can become true without v0 (D2: facts and the
    // heads of rules whose bodies are heads or facts; abar, ⊤) consecutive keys, every
    // other atom one key per 256 of its kind
    // -- and the shared copy of v_k in LEAD passes is a summary over keys (bit g = keys
    // g << kshift ..), with a per-bucket "any bit" mask on top.  The rows of every segment are bucketed (stably) by the high bits
    // g >> kb of their lead atom's group, so a LEAD pass streams only the low kb bits:
    // kb = 16 (default: a uint16 per row + a uint8 tag per 8-row octet, 2.125 B/row) or
    // kb = 8 (LP_LOAD_KEY8: a byte per row + a uint16 tag per octet, 1.25 B/row); runs of
    // one bucket padded to 8 rows.
    const bool want_keys = !p->exact && !std::getenv("LP_NO_KEYS");
    std::vector<Run> runs;
    if (want_keys) {
        std::vector<uint8_t> der((size_t)L.n_ext, 0);   // D2 (encode.cpp), abar atoms, ⊤
        for (int32_t a = 0; a < L.n; ++a) der[(size_t)a] = L.deriv2[(size_t)a];
        for (int32_t a : L.facts) der[(size_t)a] = 1;
        for (int32_t a = L.n; a < L.bot; ++a) der[(size_t)a] = 1;
        der[(size_t)L.bot] = 0;
        // derivable keys [0, nd); the underivable ones (256 atoms per key) follow, starting
        // at the next bucket boundary (a bucket = 2^16 summary groups) when that costs no
        // coarser summary, so their buckets hold nothing else
        int64_t nd = 0, nu = 0;
        for (int32_t a = 0; a < L.n_ext; ++a) (der[(size_t)a] ? nd : nu)++;
        int64_t kcap = kKeySmemBytes;
        if (opt && opt->smem_bits_cap > 0) kcap = std::min<int64_t>(kcap, opt->smem_bits_cap / 8);
        kcap = std::max<int64_t>(kcap, 16);
        auto words_for = [&](int64_t base, int s) {
            const int64_t groups = (((base + (nu + 255) / 256) - 1) >> s) + 1;
            return ((groups + 31) / 32 + 3) / 4 * 4;
        };
        int sh = 0;
        while (words_for(nd, sh) * 4 > kcap) ++sh;
        const int kb = (opt && (opt->flags & LP_LOAD_KEY8)) ? 8 : 16;   // code bits per row
        p->key_bits = kb;
        const int64_t span = (int64_t)1 << (kb + sh);   // one bucket = 2^kb groups
        int64_t nd_pad = (nd + span - 1) / span * span;
        if (words_for(nd_pad, sh) * 4 > kcap) nd_pad = nd;
        const int64_t kw = words_for(nd_pad, sh);
        const int64_t nkeys = nd_pad + (nu + 255) / 256;
        std::vector<int32_t> key((size_t)L.n_ext);
        {
            int64_t id = 0, iu = 0;
            for (int32_t a = 0; a < L.n_ext; ++a)
                key[(size_t)a] = der[(size_t)a] ? (int32_t)id++ : (int32_t)(nd_pad + (iu++ >> 8));
        }
        p->kshift = sh;
        p->ksm_words = (int32_t)kw;
        const int64_t nbuckets = (((nkeys - 1) >> sh) >> kb) + 1;
        if (nbuckets > (kb == 16 ? 32 : 32 * kBucketWords))
            return set_err(LP_E_INVALID, "internal: key bucket out of range");
        std::vector<int32_t> bucket((size_t)L.n_ext);
        for (int32_t a = 0; a < L.n_ext; ++a) bucket[(size_t)a] = (key[(size_t)a] >> sh) >> kb;
        bucket_rows(&L, bucket, 8, &runs);
        const size_t nsl = (size_t)std::max<int64_t>(L.n_slots, 8), noct = (size_t)std::max<int64_t>(L.n_slots / 8, 1);
        std::vector<uint16_t> code16(kb == 16 ? nsl : 0, 0);
        std::vector<uint8_t> code8(kb == 8 ? nsl : 0, 0);
        std::vector<uint8_t> tag8(kb == 16 ? noct : 0, 0);
        std::vector<uint16_t> tag16(kb == 8 ? noct : 0, 0);
        const int pshift = kb == 16 ? 5 : 13;
        for (const Run &r : runs) {
            const Segment &sg = L.segs[(size_t)r.seg];
            for (int64_t i = 0; i < r.rows; ++i) {
                const int64_t slot = r.slot_off + i;
                const int32_t a = L.col[(size_t)(sg.col_off + (slot - sg.slot_off))];
                const uint32_t g = (uint32_t)(key[(size_t)a] >> sh);
                if (kb == 16) code16[(size_t)slot] = (uint16_t)(g & 0xFFFF);
                else code8[(size_t)slot] = (uint8_t)(g & 0xFF);
            }
            // one tag per octet: its bucket (all 8 rows share it) and trailing padding
            const int64_t pad = r.rows_pad - r.rows;
            for (int64_t o = r.slot_off / 8; o < (r.slot_off + r.rows_pad) / 8; ++o) {
                const uint32_t t = (uint32_t)r.bucket | ((o == (r.slot_off + r.rows_pad) / 8 - 1) ? (uint32_t)pad << pshift : 0u);
                if (kb == 16) tag8[(size_t)o] = (uint8_t)t;
                else tag16[(size_t)o] = (uint16_t)t;
            }
        }
        // the run table of the live-run skip: runs tile the slot
        // space in slot order, each a multiple of 8 rows
        if (runs.size() <= (size_t)kMaxRuns && !std::getenv("LP_NO_LIVE_RUNS")) {
            std::vector<int4> rt;
            for (const Run &r : runs)
                rt.push_back(make_int4((int)(r.slot_off / 8), (int)(r.rows_pad / 8), r.bucket, 0));
            TRY(upload(p, &p->d_runs, rt));
            p->nruns = (int32_t)rt.size();
        }
        if (kb == 16) {
            uint16_t *c;
            uint8_t *t;
            TRY(upload(p, &c, code16));
            TRY(upload(p, &t, tag8));
            p->d_lead_codes = c;
            p->d_octet_tag = t;
        } else {
            uint8_t *c;
            uint16_t *t;
            TRY(upload(p, &c, code8));
            TRY(upload(p, &t, tag16));
            p->d_lead_codes = c;
            p->d_octet_tag = t;
        }
        load_mark("keys, buckets, codes");
        {   // lead-occurrence lists (pipelined LEAD passes): slots by body position 0
            std::vector<int32_t> lp((size_t)L.n_ext + 1, 0), ls;
            for (const Segment &sg : L.segs)
                for (int64_t i = 0; i < sg.count_pad; ++i) {
                    const int32_t a = L.col[(size_t)(sg.col_off + i)];
                    if (a != L.bot && a >= 0 && a < L.n_ext) lp[(size_t)a + 1]++;
                }
            for (int32_t a = 0; a < L.n_ext; ++a) lp[(size_t)a + 1] += lp[(size_t)a];
            ls.assign((size_t)std::max<int32_t>(lp[(size_t)L.n_ext], 1), 0);
            std::vector<int32_t> fo(lp.begin(), lp.end() - 1);
            for (const Segment &sg : L.segs)
                for (int64_t i = 0; i < sg.count_pad; ++i) {
                    const int32_t a = L.col[(size_t)(sg.col_off + i)];
                    if (a != L.bot && a >= 0 && a < L.n_ext) ls[(size_t)fo[(size_t)a]++] = (int32_t)(sg.slot_off + i);
                }
            TRY(upload(p, &p->d_locc_ptr, lp));
            TRY(upload(p, &p->d_locc_slot, ls));
        }
        TRY(upload(p, &p->d_key_of, key));
        std::vector<int32_t> kl;
        for (int32_t a : L.facts) kl.push_back(key[(size_t)a]);
        TRY(upload(p, &p->d_init_klist, kl));
        if (kw % 4 == 0) {   // the v_0 key summary image (LEAD passes, v0 = NULL)
            std::vector<uint32_t> ks((size_t)kw + kBucketWords, 0u);
            for (int32_t c : kl) {
                const uint32_t g = (uint32_t)c >> sh, bk = g >> kb;
                ks[g >> 5] |= 1u << (g & 31);
                ks[(size_t)kw + (bk >> 5)] |= 1u << (bk & 31);
            }
            TRY(upload(p, &p->d_init_ksum, ks));
        }
        TRY(dalloc(p, &p->d_korder, (size_t)L.n_ext + 1));
        p->lm_smem = std::max(p->lm_smem, (size_t)kw * 4);
    }

    load_mark("lead-occurrence lists");
    // exact mode, ids < 2^21: rows bucketed by (lead >> 16, head >> 16) so a LEAD pass
    // streams 16-bit lead and head planes + a 16-bit tag per 8-row octet (lead bucket |
    // head bucket << 5 | trailing padding << 10): 4.25 bytes per row instead of 8
    // (programs of >= 1 M rows: below that the stream is a few microseconds either way and
    // 8-row octets leave more threads idle than 4-row quads -- C2 measured 6 % slower)
    if (p->exact && L.n_ext <= (1 << 21) && L.n_slots >= (1 << 20) && !std::getenv("LP_NO_EXACT16")) {
        std::vector<Run> xr;
        bucket_rows_by(&L, [](int32_t lead, int32_t head) { return (lead >> 16) | ((head >> 16) << 5); }, 8, &xr);
        std::vector<uint16_t> l16((size_t)std::max<int64_t>(L.n_slots, 8), 0), h16(l16.size(), 0);
        std::vector<uint16_t> tag((size_t)std::max<int64_t>(L.n_slots / 8, 1), 0);
        for (const Run &r : xr) {
            const Segment &sg = L.segs[(size_t)r.seg];
            for (int64_t i = 0; i < r.rows; ++i) {
                const int64_t slot = r.slot_off + i;
                l16[(size_t)slot] = (uint16_t)(L.col[(size_t)(sg.col_off + (slot - sg.slot_off))] & 0xFFFF);
                h16[(size_t)slot] = (uint16_t)(L.head[(size_t)slot] & 0xFFFF);
            }
            for (int64_t o = r.slot_off / 8; o < (r.slot_off + r.rows_pad) / 8; ++o) tag[(size_t)o] = (uint16_t)r.bucket;
            tag[(size_t)((r.slot_off + r.rows_pad) / 8 - 1)] |= (uint16_t)((r.rows_pad - r.rows) << 10);
        }
        TRY(upload(p, &p->d_xlead16, l16));
        TRY(upload(p, &p->d_xhead16, h16));
        TRY(upload(p, &p->d_xtag, tag));
    }

    load_mark("exact 16-bit planes");
    // the program planes in their final row order
    if (L.has_occ) build_occ_lists(&L);
    load_mark("occurrence lists (host)");
    if (p->exact) {   // flat lead plane for exact-mode LEAD passes (one loop, no segments)
        std::vector<int32_t> l32((size_t)std::max<int64_t>(L.n_slots, 4), L.bot);
        for (const Segment &sg : L.segs)
            for (int64_t i = 0; i < sg.count_pad; ++i)
                l32[(size_t)(sg.slot_off + i)] = L.col[(size_t)(sg.col_off + i)];
        TRY(upload(p, &p->d_lead32, l32));
    }
    // armed LEAD passes (exact mode): the rows of every lead atom as records (head, L, body
    // positions 1..5, slot) -- a LEAD pass then visits only the rows whose lead atom is true
    // and whose head is not, kept in per-CTA shared-memory lists, instead of streaming the
    // lead / head planes
    // (programs of >= 1 M rows, like the 16-bit planes: below that the plane stream is a few
    // microseconds per pass and measured no slower -- C2 0.095 vs 0.100 ms armed)
    // (summary mode: the lists take the shared memory a key summary would; v_k stays in L2)
    // (normal programs: for the stable kernel's armed passes)
    if (!std::getenv("LP_NO_ARMED") &&
        (L.n_slots >= (1 << 20) || std::getenv("LP_ARMED_ALWAYS") || !L.definite)) {
        int64_t lim = (int64_t)kKeySmemBytes - (p->exact ? 4 * (int64_t)p->sm_words : 0);
        int64_t cap = std::min<int64_t>(lim / 8, p->exact ? 8192 : 16384) / 32 * 32;
        if (const char *e = std::getenv("LP_ARM_CAP")) cap = std::min<int64_t>(cap, std::atoll(e));
        if (cap >= 32) {
            std::vector<int32_t> ap((size_t)L.n_ext + 1, 0);
            for (const Segment &sg : L.segs)
                for (int64_t i = 0; i < sg.count_pad; ++i) {
                    const int32_t a = L.col[(size_t)(sg.col_off + i)];
                    if (a != L.bot) ap[(size_t)a + 1]++;
                }
            for (int32_t a = 0; a < L.n_ext; ++a) ap[(size_t)a + 1] += ap[(size_t)a];
            std::vector<int4> rec(2 * (size_t)std::max<int32_t>(ap[(size_t)L.n_ext], 1), make_int4(0, 0, 0, 0));
            std::vector<int32_t> fo(ap.begin(), ap.end() - 1);
            for (const Segment &sg : L.segs)
                for (int64_t i = 0; i < sg.count_pad; ++i) {
                    const int32_t a = L.col[(size_t)(sg.col_off + i)];
                    if (a == L.bot) continue;
                    const size_t o = (size_t)fo[(size_t)a]++;
                    const int64_t slot = sg.slot_off + i;
                    int32_t b[6] = {0, 0, 0, 0, 0, 0};
                    for (int32_t j = 1; j < sg.L && j < 6; ++j) b[j] = L.col[(size_t)(sg.col_off + (int64_t)j * sg.count_pad + i)];
                    rec[2 * o] = make_int4(L.head[(size_t)slot], sg.L, b[1], b[2]);
                    rec[2 * o + 1] = make_int4(b[3], b[4], b[5], (int32_t)slot);
                }
            TRY(upload(p, &p->d_arm_ptr, ap));
            TRY(upload(p, &p->d_arec, rec));
            p->n_records = ap[(size_t)L.n_ext];
            if (L.definite) {   // (least-model calls only run on definite programs)
                p->arm_cap = (int32_t)cap;
                p->lm_smem = std::max(p->lm_smem, (p->exact ? (size_t)p->sm_words * 4 : 0) + 8 * (size_t)cap);
            }
        }
    }
    TRY(upload(p, &p->d_segs, L.segs));
    TRY(upload(p, &p->d_col, L.col));
    TRY(upload(p, &p->d_head, L.head));
    if (L.has_occ) {
        TRY(upload(p, &p->d_occ_ptr, L.occ_ptr));
        {   // (slot, head(slot), occurrence range of that head): a firing row's head comes
            // with its slot and is queued with its own occurrence range -- two dependent
            // loads less per level
            if (L.occ_ptr[(size_t)L.n_ext] >= ((int64_t)1 << 31))
                return set_err(LP_E_INVALID, "frontier variant: more than 2^31 body entries");
            std::vector<int32_t> sh(4 * L.occ_slot.size());
            for (size_t i = 0; i < L.occ_slot.size(); ++i) {
                const size_t s = (size_t)L.occ_slot[i];   // (a placeholder entry if nnz = 0)
                const int32_t h = s < L.head.size() ? L.head[s] : 0;
                sh[4 * i] = L.occ_slot[i];
                sh[4 * i + 1] = h;
                sh[4 * i + 2] = (int32_t)L.occ_ptr[(size_t)h];
                sh[4 * i + 3] = (int32_t)L.occ_ptr[(size_t)h + 1];
            }
            TRY(upload(p, &p->d_occ_slot, sh));
            TRY(dalloc(p, &p->d_fq, (size_t)8 * ((size_t)L.n_ext + 1)));
            CK(cudaMemset(p->d_fq, 0xFF, (size_t)8 * ((size_t)L.n_ext + 1) * sizeof(int32_t)));
        }
        // the narrowest counter that holds every body length: nibbles (8 rows per word) when
        // bodies are <= 15 atoms and the segments are 8-aligned (key / 16-bit layouts), bytes
        // when <= 255, else uint32 -- the frontier's prologue re-initialises them every call
        bool al8 = true;
        for (const Segment &sg : L.segs) al8 = al8 && (sg.slot_off % 8 == 0) && (sg.count_pad % 8 == 0);
        p->cnt_bits = (L.max_body <= 15 && al8 && !std::getenv("LP_NO_NIBBLES")) ? 4 : L.max_body <= 255 ? 8 : 32;
        const size_t cw = p->cnt_bits == 4 ? ((size_t)L.n_slots + 7) / 8
                        : p->cnt_bits == 8 ? ((size_t)L.n_slots + 3) / 4 : (size_t)L.n_slots;
        TRY(dalloc(p, &p->d_cnt, std::max<size_t>(cw, 1)));
    }

    load_mark("planes + frontier uploads");
    // stable path filter: one bit per extended atom (or per 2^any_shift atoms)
    {
        int sh = 0;
        for (;; ++sh) {
            const int64_t groups = (((int64_t)L.n_ext - 1) >> sh) + 1;
            const int64_t w = ((groups + 31) / 32 + 3) / 4 * 4;
            if (w * 4 <= cap) { p->any_words = (int32_t)w; break; }
        }
        p->any_shift = sh;
        // + the "true in every guess" bits when the filter is exact and they fit
        p->st_full = sh == 0 && 2 * (int64_t)p->any_words * 4 <= cap;
        p->st_smem = (size_t)p->any_words * 4 * (p->st_full ? 2 : 1);
        // armed stable passes: CTA b owns records [b * cap, (b + 1) * cap) -- two lists of
        // cap (record, lead) pairs each after the filter bits (exact filter only)
        if (p->d_arec && !L.definite && sh == 0) {
            int64_t blocks = sms;
            if (opt && opt->grid_blocks > 0) blocks = std::min<int64_t>(blocks, opt->grid_blocks);
            const int64_t cap_st = ((p->n_records + blocks - 1) / blocks + 31) / 32 * 32;
            if (p->st_smem + 16 * (size_t)cap_st <= (size_t)kMaxSmemBytes && !std::getenv("LP_NO_ARMED_STABLE")) {
                p->st_arm_cap = (int32_t)std::max<int64_t>(cap_st, 32);
                p->st_smem += 16 * (size_t)p->st_arm_cap;
            }
        }
        TRY(dalloc(p, &p->d_any, p->any_words));
        TRY(dalloc(p, &p->d_gfull, p->any_words));
        TRY(dalloc(p, &p->d_mark, (size_t)L.n_ext));
        TRY(dalloc(p, &p->d_st_ring, 3 * ((size_t)L.n_ext + 1)));
    }

    if (!L.definite && L.k > 0 && !std::getenv("LP_NO_COMPACT_STABLE")) TRY(build_compact_stable(p));

    load_mark("stable buffers");
    CK(prepare_kernels(p->lm_smem, p->st_smem));
    if (const char *e = std::getenv("LP_CP_THREADS")) p->cp_threads = std::max(64, std::min(kThreads, std::atoi(e) / 32 * 32));
    if (p->cp_ok) {   // (small live parts: two CTAs per SM, each on its own half-words)
        p->cp_occ = std::max(1, st_compact_blocks_per_sm(0, p->cp_smem));
        p->cp_occ_search = std::max(1, st_compact_blocks_per_sm(1, p->cp_smem));
    }
    const int bl = lm_full_blocks_per_sm(p->exact, p->lm_smem);
    const int bf = lm_frontier_blocks_per_sm();
    const int bs = st_blocks_per_sm(p->st_smem);
    if (bl < 1 || bf < 1 || bs < 1) return set_err(LP_E_CUDA, "persistent kernels do not fit on an SM");
    p->grid_cap = (opt && opt->grid_blocks > 0) ? opt->grid_blocks : 0;
    auto cap_grid = [&](int b) { return p->grid_cap > 0 ? std::min(b, p->grid_cap) : b; };
    p->lm_blocks = cap_grid(sms * bl);
    {
        // a CTA handles at most 4 * threads * ceil(nq / gthreads) slots per segment, so
        // its queue never overflows (an overflow is reported, never silently dropped);
        // LEAD passes queue in both truth modes, STREAM passes in summary mode
        const int64_t gthreads = (int64_t)p->lm_blocks * kFullThreads;
        int64_t cap = 0;
        for (const Segment &sg : L.segs)
            cap += 4 * (int64_t)kFullThreads * (((sg.count_pad >> 2) + gthreads - 1) / gthreads);
        // key-mode LEAD passes: octets are dealt cyclically over all threads
        int64_t octets = 0;
        for (const Run &r : runs) octets += r.rows_pad >> 3;
        cap = std::max<int64_t>(cap, 8 * (int64_t)kFullThreads * ((octets + gthreads - 1) / gthreads));
        // overlapped LEAD passes deal octets / quads over the streaming warps only
        const int64_t sth = (int64_t)p->lm_blocks * kStreamWarps * 32;
        cap = std::max<int64_t>(cap, 8 * (int64_t)kStreamWarps * 32 * ((octets + sth - 1) / sth));
        cap = std::max<int64_t>(cap, 4 * (int64_t)kStreamWarps * 32 * (((L.n_slots >> 2) + sth - 1) / sth));
        if (cap + 8 > (1 << 28)) return set_err(LP_E_NOMEM, "candidate queue too large");
        p->qcap = (int32_t)std::max<int64_t>(cap + 8, 1024);
        // (two queues per CTA when LEAD passes are pipelined: pass k+1's candidates are
        // streamed while pass k's are verified)
        TRY(dalloc(p, &p->d_qbuf, (size_t)p->lm_blocks * p->qcap * (p->d_locc_ptr ? 2 : 1)));
    }
    p->fr_blocks = cap_grid(sms * bf);
    // one thread-block cluster for exact-mode programs whose two truth buffers fit shared
    // memory and whose flat lead / head planes a few SMs stream in a microsecond or two
    // (DESIGN.md "Cluster kernel"); the grid_blocks test hook keeps the persistent grid
    {
        const size_t cs = 3 * (size_t)p->nwords * 4;   // (three truth buffers in rotation)
        int64_t max_slots = (int64_t)1 << 16;   // (two CTAs at most: measured)
        if (const char *e = std::getenv("LP_CLUSTER_MAX_SLOTS")) max_slots = std::atoll(e);
        int64_t ent = 0;
        for (const Segment &sg : L.segs) ent += (int64_t)sg.L * sg.count_pad;
        const bool long_bodies = L.n_slots > 0 && ent > 32 * L.n_slots;   // (auto: STREAM first)
        if (p->exact && p->d_lead32 && p->grid_cap == 0 && cs <= (size_t)kMaxSmemBytes && !long_bodies &&
            L.n_slots <= max_slots && !std::getenv("LP_NO_CLUSTER")) {
            const int want = (int)std::min<int64_t>(16, std::max<int64_t>(1, (L.n_slots + 32767) / 32768));
            // one CTA and the planes fit next to the truth buffers: stage them in shared memory
            const size_t planes = 4 * (2 * (size_t)L.n_slots + (size_t)ent);
            p->cluster_stage = want == 1 && cs + planes <= (size_t)kMaxSmemBytes;
            p->cluster_smem = cs + (p->cluster_stage ? planes : 0);
            p->cluster = lm_cluster_max(want, p->cluster_smem);
            // one CTA, few rows: 512 threads (C1: 23.3 vs 25.5 us with 1024, 28.3 with 256 --
            // cheaper block barriers, still enough threads to stage the planes and stream);
            // a CTA with tens of thousands of rows keeps 1024 (paper Table 2 rows 2-4, 10-30 k
            // rules: 0.083-0.145 ms with 512 threads vs 0.064-0.104 with 1024)
            if (p->cluster == 1 && p->cl_threads == 0 && L.n_slots <= 4096) p->cl_threads = 512;
        }
    }
    if (p->cluster == 1 && !std::getenv("LP_NO_SMALL")) TRY(build_small(p));
    if (const char *e = std::getenv("LP_SMALL_THREADS")) p->small_threads = std::max(64, std::min(1024, std::atoi(e) / 32 * 32));
    p->st_blocks = cap_grid(sms * bs);
    load_mark("queues, occupancy");
    // one-cluster launches: the frontier and stable kernels of
    // programs small enough that 16 SMs carry a pass, with cluster barriers (~0.5 us) in
    // place of the 148-CTA grid barrier; the grid_blocks test hook keeps the grid
    if (p->grid_cap == 0 && !std::getenv("LP_NO_CLUSTER")) {
        // (measured on the B200: the frontier of C1 39 vs 45 us, C2 67 vs 72 us, but C3 6.1 vs
        // 4.7 ms and the C5 stable search 0.55 vs 0.21 ms -- 16 SMs do not carry those
        // passes; so only small programs, and the stable kernel stays on the grid)
        int64_t fr_max = (int64_t)1 << 20, st_max = 0;
        if (const char *e = std::getenv("LP_CLUSTER_FR_SLOTS")) fr_max = std::atoll(e);
        if (const char *e = std::getenv("LP_CLUSTER_ST_SLOTS")) st_max = std::atoll(e);
        int fr_want = 16;
        if (const char *e = std::getenv("LP_FR_CLUSTER")) fr_want = std::max(1, std::atoi(e));
        if (L.has_occ && L.n_slots <= fr_max) p->fr_cluster = cluster_size_for(0, fr_want, 0);
        if (L.n_slots <= st_max) p->st_cluster = cluster_size_for(1, 16, p->st_smem);
    }
    CK(cudaDeviceSynchronize());

    // the host copies of the big arrays are no longer needed
    std::vector<int32_t>().swap(L.col);
    std::vector<int32_t>().swap(L.head);
    std::vector<int64_t>().swap(L.occ_ptr);
    std::vector<int32_t>().swap(L.occ_slot);
    return LP_OK;
}

static void free_all(lp_program *p) {
    if (p->device >= 0) {
        cudaSetDevice(p->device);
        cudaDeviceSynchronize();
    }
    for (auto &a : p->allocs) {
        if (p->ff) p->ff(a.first, a.second, p->actx);
        else cudaFree(a.first);
    }
    p->allocs.clear();
    if (p->h_scal) cudaFreeHost(p->h_scal);
    p->h_scal = p->h_scal_dev = nullptr;
}

extern "C" lp_status lp_load(const lp_rules *rules, const lp_options *opt, lp_program **out) {
    if (!out) return set_err(LP_E_INVALID, "out is NULL");
    *out = nullptr;
    lp_program *p = new (std::nothrow) lp_program();
    if (!p) return set_err(LP_E_NOMEM, "host allocation failed");
    p->device = opt ? opt->device : 0;
    if (opt && opt->guess_cap > 0) p->guess_cap = opt->guess_cap;
    if (opt) { p->af = opt->alloc; p->ff = opt->free; p->actx = opt->alloc_ctx; }
    if ((p->af == nullptr) != (p->ff == nullptr)) {
        delete p;
        return set_err(LP_E_INVALID, "alloc and free hooks must be given together");
    }
    if (opt && (opt->flags & ~(uint32_t)(LP_LOAD_NO_FRONTIER | LP_LOAD_PAPER_LAYOUT | LP_LOAD_KEY8))) {
        delete p;
        return set_err(LP_E_INVALID, "unknown lp_options.flags bit (0x2, the former TMA ring, was removed)");
    }
    if (const char *e = std::getenv("LP_DENSE_DIV")) p->dense_div = std::max(1, std::atoi(e));
    p->env_no_pipe = std::getenv("LP_NO_PIPE") != nullptr;
    if (const char *e = std::getenv("LP_CLUSTER_THREADS")) p->cl_threads = std::atoi(e);
    if (const char *e = std::getenv("LP_FR_CLUSTER_THREADS")) p->fr_cl_threads = std::atoi(e);
    p->env_no_predict = std::getenv("LP_NO_PREDICT") != nullptr;
    p->env_no_overlap = std::getenv("LP_NO_OVERLAP") != nullptr;
    p->env_no_ksum_image = std::getenv("LP_NO_KSUM_IMAGE") != nullptr;
    p->env_no_zerocopy = std::getenv("LP_NO_ZEROCOPY") != nullptr;
    p->env_no_prefetch = std::getenv("LP_NO_PREFETCH") != nullptr;
    if (const char *e = std::getenv("LP_OVERLAP_MIN_MB")) p->overlap_min_bytes = (long long)std::atoll(e) << 20;
    if (opt && opt->derivable && !(opt->flags & LP_LOAD_PAPER_LAYOUT)) p->L.deriv_hint = opt->derivable;
    const bool occ = !(opt && (opt->flags & LP_LOAD_NO_FRONTIER));
    std::string err;
    lp_status s;
    try {
        load_mark(nullptr);
        s = encode(rules, occ && p->device >= 0, &p->L, &err,
                   opt && (opt->flags & LP_LOAD_PAPER_LAYOUT));
    } catch (const std::bad_alloc &) {
        s = LP_E_NOMEM;
        err = "host allocation failed while encoding";
    }
    if (s != LP_OK) {
        delete p;
        return set_err(s, err);
    }
    load_mark("encode (host)");
    if (p->device >= 0) {
        s = load_device(p, opt);
        if (s != LP_OK) {
            free_all(p);
            delete p;
            return s;
        }
    }
    *out = p;
    return LP_OK;
}

extern "C" void lp_free(lp_program *p) {
    if (!p) return;
    free_all(p);
    delete p;
}

extern "C" lp_status lp_info(const lp_program *p, lp_info_t *o) {
    if (!p || !o) return set_err(LP_E_INVALID, "NULL argument");
    const HostLayout &L = p->L;
    std::memset(o, 0, sizeof(*o));
    o->n_atoms = L.n_out;
    o->n_aux = L.n_aux;
    o->n_rules = L.n_rules;
    o->nnz = L.nnz;
    o->n_heads = L.n_heads;
    o->n_negated = L.k;
    o->n_free_negated = L.f;
    o->max_body = L.max_body;
    o->n_segments = (int32_t)L.segs.size();
    o->n_prime_paper = L.n_prime_paper;
    o->sparsity_eq5 = L.sparsity_eq5;
    o->device_bytes = p->dev_bytes;
    // one full θ-pass streams every body entry once (4 B, padding included) and reads +
    // writes the truth vector; heads are read only for firing rows
    int64_t col_entries = 0;
    for (const Segment &sg : L.segs) col_entries += (int64_t)sg.L * sg.count_pad;
    o->pass_bytes = 4 * col_entries + 2 * (int64_t)p->nwords * 4;
    o->lead_pass_bytes = (int64_t)lead_plane_bytes(p);
    o->stream_pass_bytes = (int64_t)stream_plane_bytes(p);
    o->truth_mode = p->exact ? 0 : 1;
    o->key_shift = p->d_lead_codes ? p->kshift : -1;
    o->summary_shift = p->shift;
    o->grid_blocks = p->lm_blocks;
    o->block_threads = kFullThreads;
    o->cluster_ctas = p->cluster;
    o->frontier_cluster_ctas = p->fr_cluster;
    o->stable_cluster_ctas = p->st_cluster;
    o->armed_list_cap = p->arm_cap;
    o->small_rows = p->small_ok ? std::max(p->sm_nr, 1) : 0;
    o->stable_compact_atoms = p->cp_ok ? p->cp_na : 0;
    o->stable_compact_rows = p->cp_ok ? p->cp_nr : 0;
    return LP_OK;
}

extern "C" lp_status lp_negated_atoms(const lp_program *p, int32_t *out) {
    if (!p) return set_err(LP_E_INVALID, "NULL program");
    if (p->L.k > 0 && !out) return set_err(LP_E_INVALID, "NULL out");
    for (int32_t j = 0; j < p->L.k; ++j) out[j] = p->L.negated[j];
    return LP_OK;
}

// ------------------------------------------------------------------------------------
// lp_least_model
// ------------------------------------------------------------------------------------

// The kernels' status word (bit flags kSt*, kernels.h) as an lp_status: an overflow is
// checked first (it is never masked by a cap or the guard); kStCapped alone is success.
static lp_status status_of(int32_t s) {
    if (s & kStOverflow) return set_err(LP_E_CUDA, "internal: candidate queue overflow");
    if (s & kStGuard) return set_err(LP_E_NOT_CONVERGED, "pass guard exceeded");
    return LP_OK;
}

// Host-pointer calls: a page-locked, mapped host buffer for the model (cudaHostAlloc /
// pinned torch tensors under unified addressing) is written by the kernel's epilogue
// itself over PCIe -- no staging buffer, no copy-engine round trip (C4 e2e 0.335 ->
// 0.320 ms).  Pageable memory: NULL (staged copy).
static void *mapped_host_ptr(const void *ptr) {
    if (!ptr) return nullptr;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
}

extern "C" lp_status lp_least_model(lp_program *p, const uint64_t *v0, uint64_t *model_out,
                                    int32_t *iters_out, const lp_run *run) {
    if (!p || !model_out || !iters_out) return set_err(LP_E_INVALID, "NULL argument");
    if (p->device < 0) return set_err(LP_E_NODEVICE, "host-only handle");
    if (!p->L.definite) return set_err(LP_E_SEMANTIC, "program is not definite");
    const HostLayout &L = p->L;
    const uint32_t flags = run ? run->flags : 0u;
    const bool dev = flags & LP_PTR_DEVICE;
    const bool frontier = flags & LP_FRONTIER;
    if (frontier && !L.has_occ)
        return set_err(LP_E_INVALID, "LP_FRONTIER on a program loaded with LP_LOAD_NO_FRONTIER");
    cudaStream_t st = run ? (cudaStream_t)run->stream : nullptr;
    CK(cudaSetDevice(p->device));
    const size_t mw = ((size_t)L.n_out + 63) / 64;
    // output window (lp_run.out_word_lo / out_word_count): model words [w0, w0 + ow)
    int64_t w0 = 0, ow = (int64_t)mw;
    if (run && run->out_word_count > 0) {
        w0 = run->out_word_lo;
        ow = run->out_word_count;
        if (w0 < 0 || w0 + ow > (int64_t)mw) return set_err(LP_E_INVALID, "output word window out of range");
    }

    const uint32_t *v0d = nullptr;
    if (v0) {
        if (dev) {
            v0d = reinterpret_cast<const uint32_t *>(v0);
        } else {   // (staged: a mapped v0 read over PCIe by the prologue measured no faster)
            if (mw) CK(cudaMemcpyAsync(p->d_v0, v0, mw * 8, cudaMemcpyHostToDevice, st));
            v0d = reinterpret_cast<const uint32_t *>(p->d_v0);
        }
    }
    int32_t *stage = nullptr;
    if (run && run->stage_out && L.n_out > 0) {
        if (dev) stage = run->stage_out;
        else {
            if (!p->d_stage) TRY(dalloc(p, &p->d_stage, (size_t)L.n_out));
            stage = p->d_stage;
        }
    }
    int32_t *pops = nullptr;
    int32_t pop_cap = 0;
    if (run && run->popcounts_out && run->popcounts_cap > 0) {
        pop_cap = run->popcounts_cap;
        if (dev) pops = run->popcounts_out;
        else {
            if (p->pops_alloc < pop_cap) {
                if (p->d_pops) dev_release(p, p->d_pops);
                TRY(dalloc(p, &p->d_pops, (size_t)pop_cap));
                p->pops_alloc = pop_cap;
            }
            pops = p->d_pops;
        }
    }

    LMParams q{};
    q.segs = p->d_segs;
    q.nseg = (int32_t)L.segs.size();
    q.n = L.n;
    q.n_out = L.n_out;
    q.n_ext_atoms = L.n_ext;
    q.n_order_cap = L.n_ext + 1;
    q.col = p->d_col;
    q.head = p->d_head;
    q.buf0 = p->d_buf0;
    q.buf1 = p->d_buf1;
    q.nwords = p->nwords;
    q.summary = p->d_summary;
    q.sm_words = p->sm_words;
    q.shift = p->shift;
    q.order = p->d_order;
    // run counters alternate between two slots: this call uses slot `par` (zeroed by
    // the previous call or at load) and zeroes the other one for the next call
    const int par = (int)(p->lm_runs & 1);
    q.tail = p->d_scal + 8 + par;
    q.tail_next = p->d_scal + 8 + (par ^ 1);
    q.status_out = p->d_scal + 10 + par;
    q.status_user = (dev && run) ? run->status_out : (!dev && p->h_scal_dev) ? p->h_scal_dev + 1 : nullptr;
    q.status_next = p->d_scal + 10 + (par ^ 1);
    q.v0 = v0d;
    q.v0_words = (int32_t)(mw * 2);
    q.factbits = p->d_factbits;
    q.init_bits = p->d_init_bits;
    q.init_list = p->d_init_list;
    q.init_klist = p->d_init_klist;
    q.init_ksum = p->env_no_ksum_image ? nullptr : p->d_init_ksum;
    q.n_init = p->n_init;
    q.top = L.top;
    void *const mout_mapped = (dev || p->env_no_zerocopy) ? nullptr : mapped_host_ptr(model_out);   // (epilogue writes over PCIe)
    unsigned long long *mout = dev ? reinterpret_cast<unsigned long long *>(model_out)
                               : mout_mapped ? reinterpret_cast<unsigned long long *>(mout_mapped) : p->d_model;
    q.model_out = mout;
    q.model_split = (mout_mapped && !frontier) ? 1 : 0;
    q.out_w0 = w0;
    q.out_wn = ow;
    q.stage = stage;
    q.pops = pops;
    q.pop_cap = pop_cap;
    q.iters_out = dev ? iters_out : p->h_scal_dev ? p->h_scal_dev : p->d_scal + 1;
    q.max_passes = L.n_ext + 2;
    q.user_cap = (run && run->max_passes > 0) ? run->max_passes : 0;
    q.occ_ptr = p->d_occ_ptr;
    q.occ_slot = p->d_occ_slot;
    q.fq = p->d_fq;
    q.cnt = p->d_cnt;
    q.cnt_bits = p->cnt_bits;
    q.dbg = debug_timing();
    q.dbg_clock = debug_clock();
    q.qbuf = p->d_qbuf;
    q.qcap = p->qcap;
    q.pass_mode = (flags & LP_FULL_STREAM) ? 2 : (flags & LP_FULL_LEAD) ? 1 : 0;
    q.dense_div = p->dense_div;
    q.predict = p->env_no_predict ? 0 : 1;
    q.prefetch = p->env_no_prefetch ? 0 : 1;
    q.n_slots = L.n_slots;
    q.cand = p->d_cand;
    q.vent = p->d_vent;
    q.overlap = p->env_no_overlap ? 0 : 1;
    q.stage_planes = p->cluster_stage ? 1 : 0;
    q.sm_blob = p->d_sm_blob;
    q.sm_blob16 = p->sm_blob16;
    q.sm_nr = p->sm_nr;
    q.sm_nnz = p->sm_nnz;
    q.cl_threads = p->cl_threads;
    q.fr_cl_threads = p->fr_cl_threads;
    q.overlap_min_bytes = p->overlap_min_bytes;
    const bool pipe = q.overlap && !(flags & LP_FULL_NO_PIPE) && !p->env_no_pipe;
    q.locc_ptr = pipe ? p->d_locc_ptr : nullptr;
    q.locc_slot = p->d_locc_slot;
    q.pbar = reinterpret_cast<uint32_t *>(p->d_scal + 24);
    q.lbar = reinterpret_cast<unsigned long long *>(p->d_scal + 28);   // (ints 28..31: 8-aligned)
    {
        long long ent = 0;
        for (const Segment &sg : L.segs) ent += (long long)sg.L * sg.count_pad;
        q.stream_entries = ent;
        // bodies this long make a LEAD verification (one sector per body entry, strided)
        // dearer than streaming: the auto schedule starts with STREAM passes
        q.auto_stream_first = (L.n_slots > 0 && ent > 32LL * L.n_slots) ? 1 : 0;
    }
    q.pcnt = p->d_scal + 16;
    unsigned long long *stats_dev = nullptr;
    if (run && run->stats_out) stats_dev = dev ? reinterpret_cast<unsigned long long *>(run->stats_out) : p->d_stats;
    if (stats_dev && frontier) {   // only the full θ-pass counts
        if (dev) CK(cudaMemsetAsync(stats_dev, 0, 6 * sizeof(uint64_t), st));
        else std::memset(run->stats_out, 0, 6 * sizeof(uint64_t));
        stats_dev = nullptr;
    }
    q.stats = stats_dev;
    // (armed LEAD passes replace the key plane: summary mode then keeps no key summary)
    q.lead_codes = (frontier || (p->d_arec && q.pass_mode != 2)) ? nullptr : p->d_lead_codes;
    q.octet_tag = p->d_octet_tag;
    q.key_bits = p->key_bits;
    q.lead32 = frontier ? nullptr : p->d_lead32;
    q.arm_ptr = p->d_arm_ptr;
    q.arec = frontier ? nullptr : p->d_arec;
    q.arm_cap = p->arm_cap;
    q.xlead16 = frontier ? nullptr : p->d_xlead16;
    q.xhead16 = p->d_xhead16;
    q.xtag = p->d_xtag;
    q.key_of = p->d_key_of;
    q.runs = p->d_runs;
    q.nruns = p->nruns;
    q.korder = p->d_korder;
    q.ksm_words = p->ksm_words;
    q.kshift = p->kshift;
    q.lead_bytes = (long long)lead_plane_bytes(p);
    q.stream_bytes = (long long)stream_plane_bytes(p);
    if (run && run->ev_begin) CK(cudaEventRecord((cudaEvent_t)run->ev_begin, st));
    // the auto schedule of an exact-mode program that fits one cluster runs there; the
    // explicit schedules (LP_FULL_STREAM / LP_FULL_LEAD / LP_FULL_NO_PIPE) keep the
    // persistent grid kernel (A/B and tests)
    const bool use_cluster = !frontier && p->cluster > 0 &&
                             !(flags & (LP_FULL_STREAM | LP_FULL_LEAD | LP_FULL_NO_PIPE));
    // (a small program's frontier call runs the small-program kernel too: it IS semi-naive,
    // by row lists instead of counters -- same model, iters, popcounts, stages)
    if (frontier && !p->small_ok) CK(launch_lm_frontier(q, p->fr_blocks, st, p->fr_cluster));
    else if (p->small_ok && (frontier || use_cluster)) CK(launch_lm_small(q, p->small_smem, st, p->small_threads));
    else if (use_cluster) CK(launch_lm_cluster(q, p->cluster, p->cluster_smem, st));
    else CK(launch_lm_full(q, p->exact, p->lm_blocks, p->lm_smem, st));
    if (run && run->ev_end) CK(cudaEventRecord((cudaEvent_t)run->ev_end, st));
    ++p->lm_runs;
    if (dev) return LP_OK;

    int32_t scal[3] = {0, 0, 0};
    if (!p->h_scal) {
        CK(cudaMemcpyAsync(scal, p->d_scal, sizeof(scal), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(scal + 2, p->d_scal + 10 + par, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    }
    if (ow && !mout_mapped) CK(cudaMemcpyAsync(model_out, p->d_model, (size_t)ow * 8, cudaMemcpyDeviceToHost, st));
    if (stage) CK(cudaMemcpyAsync(run->stage_out, stage, sizeof(int32_t) * (size_t)L.n_out,
                                  cudaMemcpyDeviceToHost, st));
    if (pops) CK(cudaMemcpyAsync(run->popcounts_out, pops, sizeof(int32_t) * (size_t)pop_cap,
                                 cudaMemcpyDeviceToHost, st));
    if (stats_dev)
        CK(cudaMemcpyAsync(run->stats_out, stats_dev, 6 * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (p->h_scal) {   // (written by the kernel's epilogue; visible once the stream is done)
        scal[1] = reinterpret_cast<volatile int32_t *>(p->h_scal)[0];
        scal[2] = reinterpret_cast<volatile int32_t *>(p->h_scal)[1];
    }
    *iters_out = scal[1];
    if (run && run->status_out) *run->status_out = scal[2];
    if (run && run->converged_out) *run->converged_out = scal[2] == 0 ? 1 : 0;
    return status_of(scal[2]);
}

// ------------------------------------------------------------------------------------
// lp_stable_models
// ------------------------------------------------------------------------------------

// The shape of the bit-sliced matrix T (n_ext rows x Wp words) for G guess columns.
static lp_status st_matrix(lp_program *p, int64_t G) {
    const int64_t W64 = (G + 63) / 64;
    if (W64 > (1 << 26)) return set_err(LP_E_INVALID, "too many guesses");
    const int32_t W = (int32_t)W64, Wp = (W + 1) / 2 * 2;
    p->W = W;
    p->Wp = Wp;
    p->G = G;
    p->stable_valid = false;
    return LP_OK;
}

// Its two buffers, allocated when something needs them: the batched kernels, or the
// expansion of a compact call's result for a readback.  (The compact kernels themselves keep
// the result as C[2W][|A*|]: C5 2.4 MB instead of 2 x 51 MB.)
static lp_status st_alloc_T(lp_program *p) {
    const size_t need = (size_t)p->L.n_ext * p->Wp;
    if (need > p->T_words_alloc) {
        if (p->d_T0) dev_release(p, p->d_T0);
        if (p->d_T1) dev_release(p, p->d_T1);
        p->d_T0 = p->d_T1 = nullptr;
        p->T_words_alloc = 0;
        TRY(dalloc(p, &p->d_T0, need));
        TRY(dalloc(p, &p->d_T1, need));
        p->T_words_alloc = need;
        p->st_dirty_ok = false;
    }
    return LP_OK;
}

// Rows of T left by the previous call: cleared by the kernel's first phase when the
// layout is unchanged (only the rows it changed), else both buffers zeroed here.
static lp_status st_clear_plan(lp_program *p, cudaStream_t st, STParams *s) {
    TRY(st_alloc_T(p));
    s->T0 = p->d_T0;
    s->T1 = p->d_T1;
    const bool full_clear = !(p->st_dirty_ok && p->st_last_Wp == p->Wp);
    p->st_last_compact = false;   // (a compact call leaves T alone; its expansion into T0 for
                                  //  a readback resets st_dirty_ok)
    if (full_clear) {   // first call, or a new matrix layout: both buffers from zero
        const size_t tbytes = (size_t)p->L.n_ext * p->Wp * sizeof(unsigned long long);
        CK(cudaMemsetAsync(p->d_T0, 0, tbytes, st));
        CK(cudaMemsetAsync(p->d_T1, 0, tbytes, st));
    }
    s->clear_rows = full_clear ? 0 : 1;
    p->st_dirty_ok = true;   // (stream order: the next call's clear runs after this one)
    p->st_last_Wp = p->Wp;
    return LP_OK;
}

static STParams st_params(lp_program *p) {
    const HostLayout &L = p->L;
    STParams s{};
    s.segs = p->d_segs;
    s.nseg = (int32_t)L.segs.size();
    s.n_ext = L.n_ext;
    s.col = p->d_col;
    s.head = p->d_head;
    s.T0 = p->d_T0;
    s.T1 = p->d_T1;
    s.Wp = p->Wp;
    s.any_init = p->d_any;
    s.gfull = p->d_gfull;
    s.use_full = p->st_full ? 1 : 0;
    s.dbg = debug_timing();
    // the flat lead plane holds extended-atom ids: usable when the any-filter is exact
    s.lead32 = (p->any_shift == 0) ? p->d_lead32 : nullptr;
    s.arm_ptr = p->d_arm_ptr;
    s.lbar = reinterpret_cast<unsigned long long *>(p->d_scal + 28);
    s.arm_cap = p->st_arm_cap;
    {   // (the ownership covers every record only if the launch has enough CTAs)
        const int64_t blocks = p->st_cluster > 0 ? p->st_cluster : p->st_blocks;
        s.arec = (p->st_arm_cap > 0 && blocks * (int64_t)p->st_arm_cap >= p->n_records) ? p->d_arec : nullptr;
    }
    s.n_slots = L.n_slots;
    s.cta_queue = (L.n_slots < (1LL << 27) && L.segs.size() <= 32) ? 1 : 0;
    s.W = p->W;
    s.G = p->G;
    s.any_words = p->any_words;
    s.any_shift = p->any_shift;
    s.order = p->d_st_ring;
    s.ring_cap = L.n_ext + 1;
    s.tail = p->d_scal + 0;
    s.pcnt = p->d_scal + 20;
    s.mark = p->d_mark;
    s.passes_out = p->d_scal + 3;
    s.status_out = p->d_scal + 2;
    s.status_user = nullptr;
    s.max_passes = L.n_ext + 2;
    return s;
}

static void st_compact_params(lp_program *p, STParams *s) {
    s->cp_blob = p->d_cp_blob;
    s->cp_blob16 = p->cp_blob16;
    s->cp_na = p->cp_na;
    s->cp_nr = p->cp_nr;
    s->cp_nnz = p->cp_nnz;
    s->cp_n0 = p->cp_n0;
    s->cp_atom = p->d_cp_atom;
    s->cp_neg = p->d_cp_neg;
    s->cp_abar = p->d_cp_abar;
    s->cp_C = p->d_cp_C;
    s->cp_pw = p->d_cp_pw;
    s->cp_done = p->d_scal + 26;
    s->cp_rp = p->d_cp_rp;
}

// the compact matrix C[W][na] of the coming compact call
static lp_status st_compact_matrix(lp_program *p) {
    const size_t cw = (size_t)p->W * p->cp_na;
    if (cw > p->cp_C_alloc) {
        if (p->d_cp_C) dev_release(p, p->d_cp_C);
        p->d_cp_C = nullptr;
        p->cp_C_alloc = 0;
        TRY(dalloc(p, &p->d_cp_C, cw));
        p->cp_C_alloc = cw;
    }
    return LP_OK;
}

// A compact call's result is the compact matrix C; the matrix / column readbacks read T0:
// zero it and scatter C into it once (T then no longer holds a batched call's dirty rows).
static lp_status st_expand_compact(lp_program *p, cudaStream_t st) {
    if (!p->st_last_compact || p->cp_expanded) return LP_OK;
    TRY(st_alloc_T(p));
    STParams s = st_params(p);
    st_compact_params(p, &s);
    s.facts = p->d_facts;   // (the all-ones rows are not in C)
    s.nfacts = p->nfacts;
    s.top = p->L.top;
    CK(cudaMemsetAsync(p->d_T0, 0, (size_t)p->L.n_ext * p->Wp * sizeof(unsigned long long), st));
    CK(launch_st_expand(s, st));
    p->cp_expanded = true;
    p->st_dirty_ok = false;
    return LP_OK;
}

extern "C" lp_status lp_stable_models(lp_program *p, const uint64_t *guesses, int64_t n_guesses,
                                      uint64_t *accepted_out, int64_t *n_accepted_out,
                                      int32_t *passes_out, const lp_run *run) {
    if (!p || !accepted_out || !n_accepted_out || !passes_out)
        return set_err(LP_E_INVALID, "NULL argument");
    if (p->device < 0) return set_err(LP_E_NODEVICE, "host-only handle");
    const HostLayout &L = p->L;
    const uint32_t flags = run ? run->flags : 0u;
    const bool dev = flags & LP_PTR_DEVICE;
    cudaStream_t st = run ? (cudaStream_t)run->stream : nullptr;
    int64_t G;
    const int64_t goff = run ? run->guess_offset : 0;
    if (goff != 0 && (guesses || goff < 0 || goff % 64))
        return set_err(LP_E_INVALID, "guess_offset needs guesses == NULL and a multiple of 64");
    if (!guesses) {
        if (L.f > p->guess_cap)
            return set_err(LP_E_CAP, "guess explosion: " + std::to_string(L.f) +
                                         " free negated atoms > guess_cap " + std::to_string(p->guess_cap));
        const int64_t all = (int64_t)1 << L.f;
        if (goff >= all) return set_err(LP_E_INVALID, "guess_offset >= 2^f");
        G = all - goff;
        if (n_guesses > 0) G = std::min(G, n_guesses);
    } else {
        if (n_guesses < 1) return set_err(LP_E_INVALID, "n_guesses < 1");
        G = n_guesses;
    }
    CK(cudaSetDevice(p->device));
    TRY(st_matrix(p, G));
    const int32_t W = p->W;
    const unsigned long long *gd = nullptr;
    if (guesses && L.k > 0) {
        if (dev) gd = reinterpret_cast<const unsigned long long *>(guesses);
        else {
            const size_t gw = (size_t)L.k * W;
            if (gw > p->guess_words_alloc) {
                if (p->d_guess) dev_release(p, p->d_guess);
                TRY(dalloc(p, &p->d_guess, gw));
                p->guess_words_alloc = gw;
            }
            CK(cudaMemcpyAsync(p->d_guess, guesses, gw * 8, cudaMemcpyHostToDevice, st));
            gd = p->d_guess;
        }
    }
    unsigned long long *acc;
    if (dev) acc = reinterpret_cast<unsigned long long *>(accepted_out);
    else {
        if ((size_t)W > p->acc_words_alloc) {
            if (p->d_acc) dev_release(p, p->d_acc);
            TRY(dalloc(p, &p->d_acc, (size_t)W));
            p->acc_words_alloc = W;
        }
        acc = p->d_acc;
    }
    long long *nacc = dev ? reinterpret_cast<long long *>(n_accepted_out)
                          : reinterpret_cast<long long *>(p->d_scal + 4);
    STParams s = st_params(p);
    if (dev) s.passes_out = passes_out;
    if (dev && run) s.status_user = run->status_out;
    s.n_atoms = L.n;
    s.k = L.k;
    s.negated = p->d_negated;
    s.negated_ext = p->d_negated_ext;
    s.free_rank = p->d_free_rank;
    s.guesses = guesses ? gd : nullptr;
    s.woff = goff / 64;
    s.facts = p->d_facts;
    s.nfacts = p->nfacts;
    s.top = L.top;
    s.any_rw = p->d_any;
    s.accepted = acc;
    s.n_accepted = nacc;
    if (p->cp_ok) {
        // compact kernel: the live sub-program in shared memory, a CTA per guess word, one
        // ordinary launch; the fixpoint matrix stays compact (C[w][A*]) until a readback
        if ((size_t)2 * W > p->cp_pw_alloc) {   // (a pass count per 32-column half-word)
            if (p->d_cp_pw) dev_release(p, p->d_cp_pw);
            TRY(dalloc(p, &p->d_cp_pw, (size_t)2 * W));
            p->cp_pw_alloc = (size_t)2 * W;
        }
        TRY(st_compact_matrix(p));
        st_compact_params(p, &s);
        p->st_last_compact = true;
        p->cp_expanded = false;
        if (run && run->ev_begin) CK(cudaEventRecord((cudaEvent_t)run->ev_begin, st));
        CK(launch_st_compact(s, std::max(1, std::min(2 * W, p->sms * p->cp_occ)), p->cp_smem, st, p->cp_threads));
    } else {
    TRY(st_clear_plan(p, st, &s));
    // ONE cooperative launch: clear, T_0, the fixpoint loop, the stability check
    if (run && run->ev_begin) CK(cudaEventRecord((cudaEvent_t)run->ev_begin, st));
    CK(launch_st_fused(s, p->st_blocks, p->st_smem, st, p->st_cluster));
    }
    if (run && run->ev_end) CK(cudaEventRecord((cudaEvent_t)run->ev_end, st));
    p->stable_valid = true;
    if (dev) return LP_OK;
    int32_t scal[6] = {0, 0, 0, 0, 0, 0};
    CK(cudaMemcpyAsync(scal, p->d_scal, sizeof(scal), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(accepted_out, acc, (size_t)W * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *passes_out = scal[3];
    int64_t na;
    std::memcpy(&na, scal + 4, sizeof(na));
    *n_accepted_out = na;
    if (run && run->status_out) *run->status_out = scal[2];
    return status_of(scal[2]);
}

// ------------------------------------------------------------------------------------
// lp_stable_search (guess-space reduction, reading R23)
// ------------------------------------------------------------------------------------

extern "C" lp_status lp_stable_search(lp_program *p, int64_t h, uint64_t seed, int32_t max_rounds,
                                      uint64_t *guesses_out, uint64_t *accepted_out,
                                      int64_t *n_accepted_out, int32_t *rounds_out,
                                      int32_t *passes_out, const lp_run *run) {
    if (!p || !accepted_out || !n_accepted_out || !rounds_out || !passes_out)
        return set_err(LP_E_INVALID, "NULL argument");
    if (p->device < 0) return set_err(LP_E_NODEVICE, "host-only handle");
    if (h < 1) return set_err(LP_E_INVALID, "h < 1");
    if (max_rounds < 1) return set_err(LP_E_INVALID, "max_rounds < 1");
    const HostLayout &L = p->L;
    const bool dev = run && (run->flags & LP_PTR_DEVICE);
    cudaStream_t st = run ? (cudaStream_t)run->stream : nullptr;
    CK(cudaSetDevice(p->device));
    TRY(st_matrix(p, h));
    const int32_t W = p->W;
    const size_t gw = std::max<size_t>((size_t)L.k * W, 1) * (p->cp_ok ? 2 : 1);   // (compact: two column buffers)
    if (gw > p->sguess_words_alloc) {
        if (p->d_sguess) dev_release(p, p->d_sguess);
        TRY(dalloc(p, &p->d_sguess, gw));
        p->sguess_words_alloc = gw;
    }
    unsigned long long *acc;
    if (dev) acc = reinterpret_cast<unsigned long long *>(accepted_out);
    else {
        if ((size_t)W > p->acc_words_alloc) {
            if (p->d_acc) dev_release(p, p->d_acc);
            TRY(dalloc(p, &p->d_acc, (size_t)W));
            p->acc_words_alloc = W;
        }
        acc = p->d_acc;
    }
    STParams s = st_params(p);
    if (p->cp_ok) TRY(st_compact_matrix(p));
    else TRY(st_clear_plan(p, st, &s));
    s.n_atoms = L.n;
    s.k = L.k;
    s.negated = p->d_negated;
    s.negated_ext = p->d_negated_ext;
    s.free_rank = p->d_free_rank;
    s.guesses = p->d_sguess;       // the round's columns
    s.gbuf = p->d_sguess;
    s.woff = 0;
    s.facts = p->d_facts;
    s.nfacts = p->nfacts;
    s.top = L.top;
    s.any_rw = p->d_any;
    s.accepted = acc;
    s.n_accepted = dev ? reinterpret_cast<long long *>(n_accepted_out)
                       : reinterpret_cast<long long *>(p->d_scal + 4);
    s.passes_out = p->d_scal + 3;   // (per round; the sum goes to passes_sum_out)
    s.seed = (unsigned long long)seed;
    s.max_rounds = max_rounds;
    s.rounds_out = dev ? rounds_out : p->d_scal + 6;
    s.passes_sum_out = dev ? passes_out : p->d_scal + 7;
    s.status_user = (dev && run) ? run->status_out : nullptr;
    if (run && run->ev_begin) CK(cudaEventRecord((cudaEvent_t)run->ev_begin, st));
    if (p->cp_ok) {   // the compact kernel's search: a CTA per guess word, a grid barrier per round
        st_compact_params(p, &s);
        p->st_last_compact = true;
        p->cp_expanded = false;
        CK(launch_st_search_compact(s, std::max(1, std::min(2 * W, p->sms * p->cp_occ_search)), p->cp_smem, st));
    } else {
        CK(launch_st_search(s, p->st_blocks, p->st_smem, st, p->st_cluster));
    }
    if (run && run->ev_end) CK(cudaEventRecord((cudaEvent_t)run->ev_end, st));
    p->stable_valid = true;
    if (guesses_out && L.k > 0)
        CK(cudaMemcpyAsync(guesses_out, p->d_sguess, (size_t)L.k * W * 8,
                           dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    if (dev) return LP_OK;
    int32_t scal[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    CK(cudaMemcpyAsync(scal, p->d_scal, sizeof(scal), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(accepted_out, acc, (size_t)W * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    int64_t na;
    std::memcpy(&na, scal + 4, sizeof(na));
    *n_accepted_out = na;
    *rounds_out = scal[6];
    *passes_out = scal[7];
    if (run && run->status_out) *run->status_out = scal[2];
    return status_of(scal[2]);
}

extern "C" lp_status lp_stable_matrix(lp_program *p, uint64_t *out, const lp_run *run) {
    if (!p || !out) return set_err(LP_E_INVALID, "NULL argument");
    if (p->device < 0) return set_err(LP_E_NODEVICE, "host-only handle");
    if (!p->stable_valid) return set_err(LP_E_INVALID, "no lp_stable_models result");
    const bool dev = run && (run->flags & LP_PTR_DEVICE);
    cudaStream_t st = run ? (cudaStream_t)run->stream : nullptr;
    CK(cudaSetDevice(p->device));
    if (p->L.n_out == 0) return LP_OK;
    TRY(st_expand_compact(p, st));
    CK(cudaMemcpy2DAsync(out, (size_t)p->W * 8, p->d_T0, (size_t)p->Wp * 8, (size_t)p->W * 8,
                         (size_t)p->L.n_out, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    if (!dev) CK(cudaStreamSynchronize(st));
    return LP_OK;
}

extern "C" lp_status lp_guess_model(lp_program *p, int64_t guess, uint64_t *model_out,
                                    const lp_run *run) {
    if (!p || !model_out) return set_err(LP_E_INVALID, "NULL argument");
    if (p->device < 0) return set_err(LP_E_NODEVICE, "host-only handle");
    if (!p->stable_valid) return set_err(LP_E_INVALID, "no lp_stable_models result");
    if (guess < 0 || guess >= p->G) return set_err(LP_E_INVALID, "guess out of range");
    const bool dev = run && (run->flags & LP_PTR_DEVICE);
    cudaStream_t st = run ? (cudaStream_t)run->stream : nullptr;
    CK(cudaSetDevice(p->device));
    TRY(st_expand_compact(p, st));
    STParams s = st_params(p);
    unsigned long long *o = dev ? reinterpret_cast<unsigned long long *>(model_out) : p->d_model;
    CK(launch_st_column(s, p->L.n_out, guess, o, st));
    if (dev) return LP_OK;
    const size_t mw = ((size_t)p->L.n_out + 63) / 64;
    if (mw) CK(cudaMemcpyAsync(model_out, p->d_model, mw * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return LP_OK;
}

// ------------------------------------------------------------------------------------
// lp_shard_combine (multi-GPU exchange step)
// ------------------------------------------------------------------------------------

extern "C" lp_status lp_shard_combine(const uint64_t *gathered, int32_t world, int64_t stride,
                                      const int64_t *word_lo, const int64_t *word_cnt,
                                      const uint64_t *v, uint64_t *v_next, int64_t n_words,
                                      int32_t *changed_out, int32_t *popcount_inout, void *stream) {
    if (!gathered || !word_lo || !word_cnt || !v || !v_next || !changed_out)
        return set_err(LP_E_INVALID, "NULL argument");
    if (world < 1 || world > kMaxRanks) return set_err(LP_E_INVALID, "world out of [1, 64]");
    if (stride < 2 || n_words < 0) return set_err(LP_E_INVALID, "stride < 2 or n_words < 0");
    ShardCombineParams q{};
    q.gathered = reinterpret_cast<const unsigned long long *>(gathered);
    q.world = world;
    q.stride = stride;
    int64_t next = 0;
    for (int32_t r = 0; r < world; ++r) {
        if (word_lo[r] != next || word_cnt[r] < 0 || word_cnt[r] > stride - 1)
            return set_err(LP_E_INVALID, "word ranges must tile [0, n_words) in rank order and fit stride - 1");
        q.word_lo[r] = word_lo[r];
        q.word_cnt[r] = word_cnt[r];
        next += word_cnt[r];
    }
    if (next != n_words) return set_err(LP_E_INVALID, "word ranges do not cover n_words");
    q.v = reinterpret_cast<const unsigned long long *>(v);
    q.v_next = reinterpret_cast<unsigned long long *>(v_next);
    q.n_words = n_words;
    q.changed = changed_out;
    q.pops = popcount_inout;
    CK(launch_shard_combine(q, (cudaStream_t)stream));
    return LP_OK;
}

extern "C" const char *lp_status_str(lp_status s) {
    switch (s) {
        case LP_OK: return "ok";
        case LP_E_INVALID: return "invalid argument";
        case LP_E_PARSE: return "parse error";
        case LP_E_SEMANTIC: return "semantic error";
        case LP_E_CAP: return "guess cap exceeded";
        case LP_E_NOMEM: return "out of memory";
        case LP_E_CUDA: return "CUDA error";
        case LP_E_NOT_CONVERGED: return "not converged";
        case LP_E_NODEVICE: return "host-only handle";
    }
    return "unknown status";
}

extern "C" const char *lp_last_error(void) { return g_err.c_str(); }

// Profiling hook, not part of include/lp.h: a device buffer of [16 passes][grid][8]
// uint64 %globaltimer stamps per CTA (pass top, stream start, stream done, verify done,
// CTA done, barrier exit) written by the next full
// θ-pass launch; NULL disables.
extern "C" void lpdbg_set_timing(void *buf) { set_debug_timing((unsigned long long *)buf); }
extern "C" void lpdbg_set_clock(int on) { set_debug_clock(on); }
