// Host-side standardiser / encoder.
//
// Turns the caller's rules into the device layout:
//   * positive form (Eq. 4): a negative literal "not a" becomes the
//     fresh atom abar_j = n + j, j = rank of a among the negated atoms (ascending);
//   * facts point at the always-true atom ⊤ = n + k (one AND-row with
//     body {⊤}), instead of the paper's diagonal a_ii = 1 (Def. 2 item 3; reading R2);
//   * every rule is one AND-row whose threshold is its (de-duplicated) body length, so
//     θ (Def. 5) is the exact integer test "all body atoms true" (reading R1);
//   * the OR-row of a multi-rule head (standardisation) is not
//     materialised: all AND-rows of a head scatter into the head's bit with an OR,
//     which is the OR-rule's T_P clause fused into the same pass;
//   * AND-rows are bucketed by body length L into position-major segments so a
//     thread streams 4 rules per int4 load with no row-pointer array.
#include <algorithm>
#include <functional>
#include <cstring>
#include <limits>

#include "lp_internal.h"

namespace lpb {

static lp_status fail(std::string *err, lp_status s, const std::string &msg) {
    if (err) *err = msg;
    return s;
}

static lp_status encode_core(const lp_rules *r, bool build_occ, HostLayout *L, std::string *err);

// Standardisation P -> P^δ, used by LP_LOAD_PAPER_LAYOUT: every head h with
// k >= 2 rules gets fresh auxiliary atoms x_1..x_k (numbered after the originals, heads in
// ascending order, rules in input order): x_i <- body(r_i) (an auxiliary fact when the
// body is empty, reading R10) and h <- x_i, i.e. the OR-row h <- x_1 ∨ ... ∨ x_k as k
// one-atom rules (the kernels OR all rules of a head).  Heads with one rule pass through.
// Iterating T over P^δ from its facts is Algorithm 1 over the paper's matrix M_{P^δ}:
// pass counts and popcount traces follow convention (A) (reading R4).
lp_status encode(const lp_rules *r, bool build_occ, HostLayout *L, std::string *err,
                 bool paper_layout) {
    if (!paper_layout || !r) {
        lp_status s = encode_core(r, build_occ, L, err);
        if (s == LP_OK) L->n_out = L->n;
        return s;
    }
    // (st_facts: the extra initial-matrix rows of Def. 8, filled in below)
    if (r->n_atoms < 0 || r->n_rules < 0) return fail(err, LP_E_INVALID, "negative n_atoms or n_rules");
    const int64_t R = r->n_rules;
    const int32_t n = r->n_atoms;
    if (R > 0 && (!r->head || !r->body_ptr)) return fail(err, LP_E_INVALID, "NULL head or body_ptr");
    for (int64_t i = 0; i < R; ++i)
        if (r->head[i] < 0 || r->head[i] >= n)
            return fail(err, LP_E_INVALID, "head out of range at rule " + std::to_string(i));
    if (R > 0 && r->body_ptr[0] != 0) return fail(err, LP_E_INVALID, "body_ptr[0] != 0");
    for (int64_t i = 0; i < R; ++i)
        if (r->body_ptr[i + 1] < r->body_ptr[i])
            return fail(err, LP_E_INVALID, "body_ptr not non-decreasing at rule " + std::to_string(i));
    if (R > 0 && r->body_ptr[R] > 0 && !r->body_atom) return fail(err, LP_E_INVALID, "NULL body_atom");
    for (int64_t j = 0; j < (R > 0 ? r->body_ptr[R] : 0); ++j)
        if (r->body_atom[j] < 0 || r->body_atom[j] >= n)
            return fail(err, LP_E_INVALID, "body atom out of range at literal " + std::to_string(j));
    std::vector<int64_t> per((size_t)n + 1, 0);
    for (int64_t i = 0; i < R; ++i) per[(size_t)r->head[i]]++;
    std::vector<int64_t> first_aux((size_t)n + 1, -1);
    int64_t naux = 0;
    for (int32_t h = 0; h < n; ++h)
        if (per[(size_t)h] >= 2) { first_aux[(size_t)h] = naux; naux += per[(size_t)h]; }
    if ((int64_t)n + naux + 2 > std::numeric_limits<int32_t>::max())
        return fail(err, LP_E_INVALID, "too many atoms after standardisation");
    const int64_t nnz_in = R > 0 ? r->body_ptr[R] : 0;
    std::vector<int32_t> head, atom;
    std::vector<int64_t> ptr{0};
    std::vector<uint8_t> neg;
    std::vector<int64_t> used((size_t)n + 1, 0);
    head.reserve((size_t)(R + naux));
    atom.reserve((size_t)(nnz_in + naux));
    for (int64_t i = 0; i < R; ++i) {
        const int32_t h = r->head[i];
        int32_t tgt = h;
        if (first_aux[(size_t)h] >= 0) {   // x_i <- body(r_i), then h <- x_i
            tgt = (int32_t)(n + first_aux[(size_t)h] + used[(size_t)h]++);
        }
        head.push_back(tgt);
        for (int64_t j = r->body_ptr[i]; j < r->body_ptr[i + 1]; ++j) {
            atom.push_back(r->body_atom[j]);
            neg.push_back(r->body_neg ? r->body_neg[j] : 0);
        }
        ptr.push_back((int64_t)atom.size());
        if (tgt != h) {
            head.push_back(h);
            atom.push_back(tgt);
            neg.push_back(0);
            ptr.push_back((int64_t)atom.size());
        }
    }
    lp_rules t{(int32_t)(n + naux), (int64_t)head.size(), head.data(), ptr.data(), atom.data(),
               r->body_neg ? neg.data() : nullptr};
    lp_status s = encode_core(&t, build_occ, L, err);
    if (s != LP_OK) return s;
    L->n_out = n;
    L->n_aux = (int32_t)naux;
    L->n_rules = R;
    // Def. 8 builds the initial guess matrix from the facts of P itself:
    // item 2 sets the row of every atom with a fact in P (even when P^δ turned that fact
    // into an auxiliary one), item 3 fixes the abar of such an atom to 0.
    std::vector<uint8_t> fact_p((size_t)n + 1, 0);
    for (int64_t i = 0; i < R; ++i)
        if (r->body_ptr[i] == r->body_ptr[i + 1]) fact_p[(size_t)r->head[i]] = 1;
    for (int32_t a = 0; a < n; ++a)
        if (fact_p[(size_t)a] && std::find(L->facts.begin(), L->facts.end(), a) == L->facts.end())
            L->st_facts.push_back(a);
    L->free_j.clear();
    for (int32_t j = 0; j < L->k; ++j)
        if (!fact_p[(size_t)L->negated[(size_t)j]]) L->free_j.push_back(j);
    L->f = (int32_t)L->free_j.size();
    return LP_OK;
}

static lp_status encode_core(const lp_rules *r, bool build_occ, HostLayout *L, std::string *err) {
    if (!r || !L) return fail(err, LP_E_INVALID, "NULL rules or output");
    const int64_t R = r->n_rules;
    const int32_t n = r->n_atoms;
    if (n < 0 || R < 0) return fail(err, LP_E_INVALID, "negative n_atoms or n_rules");
    if (R > 0 && (!r->head || !r->body_ptr))
        return fail(err, LP_E_INVALID, "NULL head or body_ptr");
    const int64_t nnz_in = R > 0 ? r->body_ptr[R] : 0;
    if (R > 0 && r->body_ptr[0] != 0) return fail(err, LP_E_INVALID, "body_ptr[0] != 0");
    for (int64_t i = 0; i < R; ++i) {
        if (r->body_ptr[i + 1] < r->body_ptr[i])
            return fail(err, LP_E_INVALID, "body_ptr not non-decreasing at rule " + std::to_string(i));
        if (r->head[i] < 0 || r->head[i] >= n)
            return fail(err, LP_E_INVALID, "head out of range at rule " + std::to_string(i));
    }
    if (nnz_in > 0 && !r->body_atom) return fail(err, LP_E_INVALID, "NULL body_atom");
    for (int64_t j = 0; j < nnz_in; ++j)
        if (r->body_atom[j] < 0 || r->body_atom[j] >= n)
            return fail(err, LP_E_INVALID, "body atom out of range at literal " + std::to_string(j));

    // ---- negated atoms, facts -----------------------------------------------------
    std::vector<uint8_t> isneg((size_t)n + 1, 0), isfact((size_t)n + 1, 0);
    if (r->body_neg)
        for (int64_t j = 0; j < nnz_in; ++j)
            if (r->body_neg[j]) isneg[r->body_atom[j]] = 1;
    for (int64_t i = 0; i < R; ++i)
        if (r->body_ptr[i] == r->body_ptr[i + 1]) isfact[r->head[i]] = 1;
    std::vector<int32_t> jof((size_t)n + 1, -1);
    int32_t k = 0;
    for (int32_t a = 0; a < n; ++a)
        if (isneg[a]) { jof[a] = k++; L->negated.push_back(a); }
    if ((int64_t)n + k + 2 > std::numeric_limits<int32_t>::max())
        return fail(err, LP_E_INVALID, "too many atoms for int32 ids");
    for (int32_t j = 0; j < k; ++j)
        if (!isfact[L->negated[j]]) L->free_j.push_back(j);
    for (int32_t a = 0; a < n; ++a)
        if (isfact[a]) L->facts.push_back(a);

    L->n = n;
    L->k = k;
    L->f = (int32_t)L->free_j.size();
    L->top = n + k;
    L->bot = n + k + 1;
    L->n_ext = n + k + 2;
    L->n_rules = R;
    L->definite = (k == 0);

    // ---- rules per head (statistics, and the derivability sets below)
    std::vector<int32_t> per_head((size_t)n + 1, 0);
    for (int64_t i = 0; i < R; ++i) per_head[r->head[i]]++;

    // ---- per-rule de-duplicated extended bodies -----------------------------------
    std::vector<int32_t> ext((size_t)std::max<int64_t>(nnz_in, 1));
    std::vector<int32_t> len((size_t)std::max<int64_t>(R, 1));
    std::vector<int32_t> tmp;
    int64_t pos = 0;
    int32_t maxL = 0;
    for (int64_t i = 0; i < R; ++i) {
        const int64_t s = r->body_ptr[i], e = r->body_ptr[i + 1];
        const int64_t start = pos;
        if (e - s <= 16) {
            for (int64_t j = s; j < e; ++j) {
                int32_t a = r->body_atom[j];
                int32_t x = (r->body_neg && r->body_neg[j]) ? n + jof[a] : a;
                bool dup = false;
                for (int64_t q = start; q < pos; ++q)
                    if (ext[q] == x) { dup = true; break; }
                if (!dup) ext[pos++] = x;
            }
        } else {
            tmp.clear();
            for (int64_t j = s; j < e; ++j) {
                int32_t a = r->body_atom[j];
                tmp.push_back((r->body_neg && r->body_neg[j]) ? n + jof[a] : a);
            }
            std::sort(tmp.begin(), tmp.end());
            tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
            for (int32_t x : tmp) ext[pos++] = x;
        }
        int64_t l = pos - start;
        if (l > std::numeric_limits<int32_t>::max()) return fail(err, LP_E_INVALID, "body too long");
        len[i] = (int32_t)l;
        if ((int32_t)l > maxL) maxL = (int32_t)l;
    }
    L->max_body = maxL;

    // ---- a static over-approximation of the atoms that can become true from the facts
    // alone: D1 = heads ∪ facts, D2 = facts ∪ {head(r) : body(r) ⊆ D1} (abar atoms count
    // as true: the guesses set them).  Two unfoldings only -- a layout heuristic, computed
    // from the program, never from v0: an atom outside D2 is true only if v0 says so.
    // It picks each row's lead atom here and the fine/coarse key groups at load.
    L->deriv2.assign((size_t)n, 0);
    if (L->deriv_hint) {   // the caller's D2 (lp_options.derivable: e.g. of the whole program
                           // when this one is a head-range shard of it)
        for (int32_t a = 0; a < n; ++a) L->deriv2[(size_t)a] = L->deriv_hint[a] ? 1 : 0;
    } else {
        auto in_d1 = [&](int32_t x) { return x >= n || per_head[(size_t)x] || isfact[(size_t)x]; };
        int64_t q = 0;
        for (int64_t i = 0; i < R; ++i) {
            bool all = true;
            for (int64_t j = q; j < q + len[i] && all; ++j) all = in_d1(ext[j]);
            if (all) L->deriv2[(size_t)r->head[i]] = 1;   // (facts: empty body)
            q += len[i];
        }
    }
    for (int64_t i = 0; i < R; ++i)   // (facts are always derivable)
        if (len[i] == 0) L->deriv2[(size_t)r->head[i]] = 1;
    // lead atom (body position 0, the one the full θ-pass streams first and tests before
    // anything else is loaded): the first body atom outside D2 if there is one, else the
    // input order is kept.  The AND is order-free, so this changes how many rows need a
    // second look, never a result.
    {
        int64_t q = 0;
        for (int64_t i = 0; i < R; ++i) {
            for (int64_t j = q; j < q + len[i]; ++j) {
                const int32_t x = ext[j];
                if (x < n && !L->deriv2[(size_t)x]) {
                    std::swap(ext[q], ext[j]);
                    break;
                }
            }
            q += len[i];
        }
    }
    int64_t n_fact_rules = 0;
    for (int64_t i = 0; i < R; ++i) n_fact_rules += len[i] == 0;

    // ---- statistics ----------------------------------------------------------------
    {
        int64_t heads = 0, aux = 0;
        for (int32_t a = 0; a < n; ++a) {
            if (per_head[a]) ++heads;
            if (per_head[a] >= 2) aux += per_head[a];
        }
        L->n_heads = heads;
        L->n_prime_paper = (int64_t)n + k + aux;
        L->sparsity_eq5 = n == 0 ? 1.0 : 1.0 - (double)nnz_in / ((double)n * (double)n);
    }

    // ---- segments by body length ---------------------------------------------------
    // A fact is the AND-row {⊤} (reading R2).  Its head is put into v_0 by the init
    // kernel and the row can never add anything after that, so it is not stored in the
    // pass segments; nnz still counts its ⊤ entry.
    std::vector<int64_t> cnt((size_t)maxL + 1, 0);
    for (int64_t i = 0; i < R; ++i)
        if (len[i]) cnt[len[i]]++;
    std::vector<int32_t> segof((size_t)maxL + 1, -1);
    int64_t col_off = 0, slot_off = 0, nnz = 0;
    for (int32_t l = 1; l <= maxL; ++l) {
        if (!cnt[l]) continue;
        Segment sg{};
        sg.L = l;
        sg.count = cnt[l];
        sg.count_pad = (cnt[l] + 3) / 4 * 4;
        sg.col_off = col_off;
        sg.slot_off = slot_off;
        col_off += (int64_t)l * sg.count_pad;
        slot_off += sg.count_pad;
        nnz += (int64_t)l * sg.count;
        segof[l] = (int32_t)L->segs.size();
        L->segs.push_back(sg);
    }
    if (slot_off > std::numeric_limits<int32_t>::max())
        return fail(err, LP_E_INVALID, "too many rules for int32 slots");
    L->nnz = nnz + n_fact_rules;
    L->n_slots = slot_off;
    L->col.assign((size_t)col_off, L->bot);
    L->head.assign((size_t)slot_off, L->bot);
    std::vector<int64_t> fillc(L->segs.size(), 0);
    pos = 0;
    for (int64_t i = 0; i < R; ++i) {
        const int32_t l = len[i];
        if (l == 0) continue;   // fact: its head is in v_0 already (row {⊤} never adds anything)
        const Segment &sg = L->segs[segof[l]];
        const int64_t slot = fillc[segof[l]]++;
        int32_t *c = L->col.data() + sg.col_off + slot;
        for (int32_t j = 0; j < l; ++j) c[(int64_t)j * sg.count_pad] = ext[pos + j];
        pos += l;
        L->head[sg.slot_off + slot] = r->head[i];
    }

    // the transposed occurrence lists (frontier variant) are built by the loader after
    // the final row order is fixed (build_occ_lists)
    L->has_occ = build_occ;
    return LP_OK;
}

// Transposed occurrence lists over extended atoms (frontier variant, SURVEY.md §8(a)
// a6): occ_slot[occ_ptr[a] .. occ_ptr[a+1]) = the slots whose body contains a.  Padding
// rows (body ⊥) are skipped.
void build_occ_lists(HostLayout *L) {
    L->occ_ptr.assign((size_t)L->n_ext + 1, 0);
    for (const Segment &sg : L->segs)
        for (int32_t j = 0; j < sg.L; ++j) {
            const int32_t *c = L->col.data() + sg.col_off + (int64_t)j * sg.count_pad;
            for (int64_t i = 0; i < sg.count_pad; ++i)
                if (c[i] != L->bot) L->occ_ptr[(size_t)c[i] + 1]++;
        }
    for (int32_t a = 0; a < L->n_ext; ++a) L->occ_ptr[(size_t)a + 1] += L->occ_ptr[(size_t)a];
    L->occ_slot.assign((size_t)std::max<int64_t>(L->occ_ptr[(size_t)L->n_ext], 1), 0);
    std::vector<int64_t> fo(L->occ_ptr.begin(), L->occ_ptr.end() - 1);
    for (const Segment &sg : L->segs)
        for (int32_t j = 0; j < sg.L; ++j) {
            const int32_t *c = L->col.data() + sg.col_off + (int64_t)j * sg.count_pad;
            for (int64_t i = 0; i < sg.count_pad; ++i)
                if (c[i] != L->bot) L->occ_slot[(size_t)fo[(size_t)c[i]]++] = (int32_t)(sg.slot_off + i);
        }
}

// Stable reorder of the rows of every segment by bucket(lead atom); every bucket's run
// is padded with ⊥ rows to a multiple of `align` rows (the AND-rows of a segment are in
// no particular order, so this changes no result).  Segment offsets are recomputed; the
// run table lists (segment, bucket, first slot, real rows, padded rows) in slot order.
void bucket_rows(HostLayout *L, const std::vector<int32_t> &bucket_of_atom, int align,
                 std::vector<Run> *runs) {
    bucket_rows_by(L, [&](int32_t lead, int32_t) { return bucket_of_atom[(size_t)lead]; }, align, runs);
}

void bucket_rows_by(HostLayout *L, const std::function<int32_t(int32_t, int32_t)> &bucket_of,
                    int align, std::vector<Run> *runs) {
    std::vector<Segment> segs;
    std::vector<int32_t> col, head;
    int64_t col_off = 0, slot_off = 0;
    runs->clear();
    // pass 1: sizes
    std::vector<std::vector<int64_t>> counts(L->segs.size());
    int32_t nb = 0;
    for (const Segment &sg : L->segs) {
        const int32_t *c0 = L->col.data() + sg.col_off;
        for (int64_t i = 0; i < sg.count_pad; ++i)
            if (c0[i] != L->bot) nb = std::max(nb, bucket_of(c0[i], L->head[(size_t)(sg.slot_off + i)]) + 1);
    }
    for (size_t s = 0; s < L->segs.size(); ++s) {
        const Segment &sg = L->segs[s];
        counts[s].assign((size_t)nb, 0);
        const int32_t *c0 = L->col.data() + sg.col_off;
        for (int64_t i = 0; i < sg.count_pad; ++i)
            if (c0[i] != L->bot) counts[s][(size_t)bucket_of(c0[i], L->head[(size_t)(sg.slot_off + i)])]++;
        Segment ns = sg;
        ns.count = 0;
        ns.count_pad = 0;
        for (int32_t b = 0; b < nb; ++b) {
            const int64_t n = counts[s][(size_t)b];
            if (!n) continue;
            const int64_t np = (n + align - 1) / align * align;
            runs->push_back(Run{(int32_t)s, b, slot_off + ns.count_pad, n, np});
            ns.count += n;
            ns.count_pad += np;
        }
        ns.col_off = col_off;
        ns.slot_off = slot_off;
        col_off += (int64_t)ns.L * ns.count_pad;
        slot_off += ns.count_pad;
        segs.push_back(ns);
    }
    col.assign((size_t)col_off, L->bot);
    head.assign((size_t)slot_off, L->bot);
    // pass 2: stable scatter (bucket runs in ascending bucket order inside each segment)
    size_t ri = 0;
    for (size_t s = 0; s < L->segs.size(); ++s) {
        const Segment &sg = L->segs[s];
        const Segment &ns = segs[s];
        std::vector<int64_t> next((size_t)nb, -1);
        for (; ri < runs->size() && (*runs)[ri].seg == (int32_t)s; ++ri)
            next[(size_t)(*runs)[ri].bucket] = (*runs)[ri].slot_off - ns.slot_off;
        const int32_t *c0 = L->col.data() + sg.col_off;
        for (int64_t i = 0; i < sg.count_pad; ++i) {
            if (c0[i] == L->bot) continue;
            const int64_t d = next[(size_t)bucket_of(c0[i], L->head[(size_t)(sg.slot_off + i)])]++;
            for (int32_t j = 0; j < sg.L; ++j)
                col[(size_t)(ns.col_off + (int64_t)j * ns.count_pad + d)] =
                    L->col[(size_t)(sg.col_off + (int64_t)j * sg.count_pad + i)];
            head[(size_t)(ns.slot_off + d)] = L->head[(size_t)(sg.slot_off + i)];
        }
    }
    L->segs.swap(segs);
    L->col.swap(col);
    L->head.swap(head);
    L->n_slots = slot_off;
}

}  // namespace lpb
