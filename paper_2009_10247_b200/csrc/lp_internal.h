// Internal structures shared by the host encoder (encode.cpp), the kernels
// (kernels.cu) and the ABI glue (abi.cu).  Not part of the public ABI.
#pragma once
#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "../../include/lp.h"

namespace lpb {

// One body-length bucket of AND-rows.
// Rule slot i (0 <= i < count_pad) of the segment has body atoms
//   col[col_off + j * count_pad + i]   for j = 0..L-1    (position-major, coalesced)
// and head head[slot_off + i].  Slots count..count_pad-1 are padding rules whose body
// is the always-false atom ⊥ and whose head is ⊥ (they never fire).
struct Segment {
    int32_t L;
    int32_t pad_;
    int64_t count;
    int64_t count_pad;   // multiple of 4 (int4 loads of 4 rules per position)
    int64_t col_off;     // in int32 elements, multiple of 4
    int64_t slot_off;    // in rule slots, multiple of 4
};

// Host-side result of standardisation + encoding.
struct HostLayout {
    int32_t n = 0;        // atoms of the encoded program (originals + P^δ auxiliaries)
    int32_t n_out = 0;    // atoms the caller sees (v0, models, stages): the originals
    int32_t n_aux = 0;    // LP_LOAD_PAPER_LAYOUT: auxiliary atoms n_out .. n-1
    int32_t k = 0;        // negated atoms (abar_j = n + j)
    int32_t f = 0;        // free negated atoms (not facts)
    int32_t top = 0;      // ⊤ = n + k  (always true; body of every fact)
    int32_t bot = 0;      // ⊥ = n + k + 1 (always false; padding)
    int32_t n_ext = 0;    // n + k + 2
    int64_t n_rules = 0;
    int64_t nnz = 0;      // real body entries (after dedupe, facts count 1 for ⊤)
    int64_t n_heads = 0;
    int64_t n_prime_paper = 0;
    int32_t max_body = 0;
    double sparsity_eq5 = 1.0;
    bool definite = true;

    std::vector<Segment> segs;
    std::vector<int32_t> col;       // all segments, position-major
    std::vector<int32_t> head;      // per slot
    int64_t n_slots = 0;

    std::vector<int32_t> facts;     // distinct atoms with a fact rule (in the encoded program)
    std::vector<uint8_t> deriv2;    // [n] atom in D2 (encode.cpp): may become true from the facts
    const uint8_t *deriv_hint = nullptr;   // [n] caller's D2 (lp_options.derivable), or NULL
    std::vector<int32_t> st_facts;  // LP_LOAD_PAPER_LAYOUT: atoms with a fact in P whose
                                    // fact became an auxiliary one (Def. 8 item 2 rows)
    std::vector<int32_t> negated;   // k ascending atom ids
    std::vector<int32_t> free_j;    // indices j of the free negated atoms (ascending)

    // transposed occurrence lists over extended atoms (frontier variant)
    bool has_occ = false;
    std::vector<int64_t> occ_ptr;   // [n_ext + 1]
    std::vector<int32_t> occ_slot;  // [nnz]
};

// A run of rows of one segment whose lead atoms share a bucket (key-mode LEAD passes).
struct Run {
    int32_t seg;
    int32_t bucket;
    int64_t slot_off;   // first slot (multiple of the alignment)
    int64_t rows;       // real rows
    int64_t rows_pad;   // rows incl. ⊥ padding (multiple of the alignment)
};

// encode.cpp
lp_status encode(const lp_rules *r, bool build_occ, HostLayout *out, std::string *err,
                 bool paper_layout = false);
void build_occ_lists(HostLayout *L);
void bucket_rows(HostLayout *L, const std::vector<int32_t> &bucket_of_atom, int align,
                 std::vector<Run> *runs);
// the same with the bucket a function of (lead atom, head) of a row
void bucket_rows_by(HostLayout *L, const std::function<int32_t(int32_t, int32_t)> &bucket_of,
                    int align, std::vector<Run> *runs);

}  // namespace lpb
