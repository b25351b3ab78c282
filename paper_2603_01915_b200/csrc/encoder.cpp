// Byte-identical CSR-dtANS encoder (host, C++17, multithreaded).
//
// Restates the reference encoder so the container bytes match exactly:
//   encode_matrix            container.py:126-204
//   matrix_deltas            sparse.py:289-299 ; value_patterns sparse.py:302-309
//   _distribution_from_array container.py:112-114 (ascending unique + counts)
//   quantize / _allocate     entropy.py:201-321
//   build_tables/from_slots  entropy.py:351-436 ; pad_symbol entropy.py:392-401
//   dtans_encode             codec.py:241-368 (base pass, backward digit pass)
//   interleave_warp          container.py:254-317 (lockstep event order)
//   _tables_block            container.py:604-625 (slot record layout)
// The quantizer is the only floating-point step: it uses glibc log2 (what
// CPython's math.log2 calls) and is compiled with -ffp-contract=off so every
// product and sum is rounded exactly as in the reference.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <new>
#include <queue>
#include <string>
#include <thread>
#include <vector>

#include "common.h"
#include "encoder_internal.h"

namespace dtans {

static thread_local std::string g_last_error;
void set_error_text(const char *msg) { g_last_error = msg; }

namespace {

// ----------------------------------------------------------------------------
// Distributions (container.py:112-114): sorted unique symbols with counts.


static void rle_sorted(const uint64_t *a, size_t n, std::vector<uint64_t> &s,
                       std::vector<int64_t> &c)
{
    size_t i = 0;
    while (i < n) {
        size_t j = i + 1;
        while (j < n && a[j] == a[i]) j++;
        s.push_back(a[i]);
        c.push_back((int64_t)(j - i));
        i = j;
    }
}

// Merge per-chunk (sym, cnt) runs (each ascending) into one ascending list.
static Dist merge_runs(std::vector<std::vector<uint64_t>> &syms,
                       std::vector<std::vector<int64_t>> &cnts)
{
    // pairwise merge until one list remains
    while (syms.size() > 1) {
        std::vector<std::vector<uint64_t>> ns;
        std::vector<std::vector<int64_t>> nc;
        for (size_t p = 0; p + 1 < syms.size(); p += 2) {
            auto &as = syms[p], &bs = syms[p + 1];
            auto &ac = cnts[p], &bc = cnts[p + 1];
            std::vector<uint64_t> os;
            std::vector<int64_t> oc;
            os.reserve(as.size() + bs.size());
            oc.reserve(as.size() + bs.size());
            size_t i = 0, j = 0;
            while (i < as.size() || j < bs.size()) {
                if (j >= bs.size() || (i < as.size() && as[i] < bs[j])) {
                    os.push_back(as[i]); oc.push_back(ac[i]); i++;
                } else if (i >= as.size() || bs[j] < as[i]) {
                    os.push_back(bs[j]); oc.push_back(bc[j]); j++;
                } else {
                    os.push_back(as[i]); oc.push_back(ac[i] + bc[j]); i++; j++;
                }
            }
            ns.push_back(std::move(os));
            nc.push_back(std::move(oc));
        }
        if (syms.size() % 2) {
            ns.push_back(std::move(syms.back()));
            nc.push_back(std::move(cnts.back()));
        }
        syms.swap(ns);
        cnts.swap(nc);
    }
    Dist d;
    if (!syms.empty()) {
        d.sym = std::move(syms[0]);
        d.cnt = std::move(cnts[0]);
    }
    for (int64_t c : d.cnt) d.total += c;
    return d;
}

// ----------------------------------------------------------------------------
// quantize (entropy.py:223-321) with _allocate (entropy.py:201-220).

struct Quant {
    std::vector<int32_t> mult;  // per distinct symbol; 0 = escaped
    int32_t esc_mult = 0;
    int32_t esc_slots = 0;
};

struct Eval {
    bool ok = false;
    double cost = 0.0;
    int64_t kk = 0;
    std::vector<int32_t> retained_mult;  // aligned with eligible[:kk]
    int32_t esc_mult = 0, esc_slots = 0;
};

struct HeapItem {
    double key;    // -count, then -gain (entropy.py:211,218-219)
    int64_t rank;  // tie-break: smaller rank first
    int64_t i;
    bool operator>(const HeapItem &o) const
    {
        if (key != o.key) return key > o.key;
        if (rank != o.rank) return rank > o.rank;
        return i > o.i;
    }
};

class Quantizer {
  public:
    Quantizer(const std::vector<int64_t> &counts, const std::vector<char> &never,
              int32_t k, int32_t m, int32_t raw)
        : counts_(counts), k_(k), m_(m), raw_(raw)
    {
        const int64_t n = (int64_t)counts.size();
        total_ = 0;
        for (int64_t c : counts) total_ += c;
        // sorted(range(n), key=lambda i: (-counts[i], i)) minus never_retain:
        // only the first min(n_eligible, k) entries are ever retained, so
        // only the first top = k + |never| + 1 of that order are built: the
        // top-th largest count (selection on a contiguous copy), every index
        // above it, then the tied ones in index order (the order is total).
        int64_t n_never = 0;
        for (int64_t i = 0; i < n; i++) n_never += never[i] ? 1 : 0;
        n_eligible_ = n - n_never;
        const int64_t top = std::min<int64_t>(n, (int64_t)k + n_never + 1);
        std::vector<int64_t> order;
        order.reserve((size_t)top);
        if (top > 0) {
            std::vector<int64_t> cs(counts.begin(), counts.end());
            std::nth_element(cs.begin(), cs.begin() + (top - 1), cs.end(), std::greater<int64_t>());
            const int64_t cth = cs[top - 1];
            for (int64_t i = 0; i < n; i++)
                if (counts[i] > cth) order.push_back(i);
            for (int64_t i = 0; i < n && (int64_t)order.size() < top; i++)
                if (counts[i] == cth) order.push_back(i);
            std::sort(order.begin(), order.end(),
                      [&](int64_t a, int64_t b) { return counts[a] != counts[b] ? counts[a] > counts[b] : a < b; });
        }
        for (int64_t i : order)
            if (!never[i]) eligible_.push_back(i);
        prefix_.assign(eligible_.size() + 1, 0);
        for (size_t j = 0; j < eligible_.size(); j++)
            prefix_[j + 1] = prefix_[j] + counts[eligible_[j]];
        logk_ = std::log2((double)k);
        lg_.resize((size_t)std::max(m, 2) + 2);
        for (size_t x = 1; x < lg_.size(); x++) lg_[x] = std::log2((double)x);
    }

    // _allocate(counts, ranks, slots, cap) -> mult, leftover
    void allocate(const std::vector<int64_t> &ec, std::vector<int32_t> &mult,
                  int64_t &left) const
    {
        const int64_t n = (int64_t)ec.size();
        mult.assign(n, 1);
        left = (int64_t)k_ - n;
        std::vector<HeapItem> heap;
        if (m_ > 1) {
            heap.reserve(n);
            for (int64_t i = 0; i < n; i++) heap.push_back({-(double)ec[i], i, i});
        }
        std::priority_queue<HeapItem, std::vector<HeapItem>, std::greater<HeapItem>> pq(
            std::greater<HeapItem>(), std::move(heap));
        while (left > 0 && !pq.empty()) {
            HeapItem it = pq.top();
            pq.pop();
            const int64_t i = it.i;
            mult[i] += 1;
            left -= 1;
            if (mult[i] < m_) {
                const double diff = lg_[mult[i] + 1] - lg_[mult[i]];
                const double gain = (double)ec[i] * diff;
                pq.push({-gain, i, i});
            }
        }
    }

    Eval evaluate(int64_t kk) const
    {
        Eval e;
        e.kk = kk;
        const int64_t escaped = total_ - prefix_[kk];
        const bool escape_needed = escaped > 0;
        const int64_t n_ent = kk + (escape_needed ? 1 : 0);
        if (n_ent > k_ || (n_ent == 0 && total_ > 0)) return e;
        if (n_ent == 0) {
            e.ok = true;
            e.cost = 0.0;
            e.esc_mult = std::min(m_, k_);
            e.esc_slots = k_;
            return e;
        }
        std::vector<int64_t> ec(n_ent);
        for (int64_t j = 0; j < kk; j++) ec[j] = counts_[eligible_[j]];
        if (escape_needed) ec[kk] = escaped;
        std::vector<int32_t> mult;
        int64_t leftover;
        allocate(ec, mult, leftover);
        int64_t esc_mult = escape_needed ? mult[kk] : 0;
        if (leftover > 0 && !escape_needed) {
            if (kk + 1 > k_) return e;
            esc_mult = std::min<int64_t>(m_, leftover);
            leftover -= esc_mult;
        }
        const int64_t esc_slots = esc_mult ? (esc_mult + leftover) : 0;
        if (esc_mult == 0 && leftover > 0) return e;
        double cost = 0.0;
        for (int64_t j = 0; j < kk; j++) {
            const double t = logk_ - lg_[mult[j]];
            cost += (double)ec[j] * t;
        }
        if (escaped > 0) {
            const double t = (logk_ - lg_[esc_mult]) + (double)raw_;
            cost += (double)escaped * t;
        }
        e.ok = true;
        e.cost = cost;
        e.retained_mult.assign(mult.begin(), mult.begin() + kk);
        e.esc_mult = (int32_t)esc_mult;
        e.esc_slots = (int32_t)esc_slots;
        return e;
    }

    // best_in(lo, hi, step): scan kk downward, strict < keeps the first best
    bool best_in(int64_t lo, int64_t hi, int64_t step, Eval &best) const
    {
        bool have = false;
        for (int64_t kk = hi; kk >= lo; kk -= step) {
            Eval r = evaluate(kk);
            if (r.ok && (!have || r.cost < best.cost)) {
                best = std::move(r);
                have = true;
            }
        }
        return have;
    }

    bool run(Quant &q) const
    {
        const int64_t kExhaustive = 96;  // entropy.py:198
        const int64_t kk_hi = std::min<int64_t>(n_eligible_, k_);
        Eval best;
        bool have;
        if (kk_hi + 1 <= kExhaustive) {
            have = best_in(0, kk_hi, 1, best);
        } else {
            int64_t lo = 0, hi = kk_hi;
            while (hi - lo + 1 > kExhaustive) {
                const int64_t step = std::max<int64_t>(1, (hi - lo) / 32);
                Eval found;
                if (!best_in(lo, hi, step, found)) break;
                const int64_t center = found.kk;
                lo = std::max(lo, center - 2 * step);
                hi = std::min(hi, center + 2 * step);
            }
            have = best_in(lo, hi, 1, best);
        }
        if (!have) return false;
        q.mult.assign(counts_.size(), 0);
        for (int64_t j = 0; j < best.kk; j++) q.mult[eligible_[j]] = best.retained_mult[j];
        q.esc_mult = best.esc_mult;
        q.esc_slots = best.esc_slots;
        return true;
    }

  private:
    const std::vector<int64_t> &counts_;
    int32_t k_, m_, raw_;
    int64_t total_;
    std::vector<int64_t> eligible_;  // the first min(n_eligible, k + 1) in (-count, index) order
    int64_t n_eligible_ = 0;
    std::vector<int64_t> prefix_;
    double logk_;
    std::vector<double> lg_;
};

// ----------------------------------------------------------------------------
// Coding tables (entropy.py:333-436) + encoder-side inverse maps.



static bool build_domain(const Dist &dist, const Quant &q, const uint32_t *perm,
                         int32_t k, int payload_words, Domain &D)
{
    // canonical entries (entropy.py:413-424)
    struct Ent { int32_t id; int32_t d; int32_t b; };  // id -1 = ESCAPE
    std::vector<Ent> entries;
    entries.reserve(k);
    int32_t nret = 0;
    std::vector<uint64_t> ret_sym;
    for (size_t i = 0; i < dist.sym.size(); i++) {
        const int32_t x = q.mult[i];
        if (x > 0) {
            for (int32_t d = 0; d < x; d++) entries.push_back({nret, d, x});
            ret_sym.push_back(dist.sym[i]);
            D.id_base.push_back((uint16_t)x);
            nret++;
        }
    }
    if (q.esc_slots) {
        const int32_t e = q.esc_mult;
        for (int32_t d = 0; d < e; d++) entries.push_back({-1, d, e});
        int32_t filler = q.esc_slots - e;
        while (filler > 0) {
            const int32_t run = std::min(e, filler);
            for (int32_t d = 0; d < run; d++) entries.push_back({-1, d, run});
            filler -= run;
        }
    }
    if ((int32_t)entries.size() != k) return false;
    std::vector<Ent> placed(k);
    if (perm) {
        std::vector<char> seen(k, 0);
        for (int32_t pos = 0; pos < k; pos++) {
            const uint32_t p = perm[pos];
            if (p >= (uint32_t)k || seen[p]) return false;
            seen[p] = 1;
            placed[p] = entries[pos];
        }
    } else {
        placed = entries;
    }
    D.sym.assign(k, 0);
    D.dig.assign(k, 0);
    D.base.assign(k, 0);
    D.esc.assign(k, 0);
    D.id_off.assign(nret + 1, 0);
    for (int32_t i = 0; i < nret; i++) D.id_off[i + 1] = D.id_off[i] + D.id_base[i];
    D.slot_by_digit.assign(D.id_off[nret], 0);
    D.esc_base = 0;
    for (int32_t j = 0; j < k; j++)
        if (placed[j].id < 0) D.esc_base = std::max(D.esc_base, placed[j].b);
    D.esc_slot.assign(256 + 1, 0xFFFF);
    int32_t best_b = 0;
    for (int32_t j = 0; j < k; j++) {
        const Ent &e = placed[j];
        D.dig[j] = (uint8_t)e.d;
        D.base[j] = (uint16_t)e.b;
        if (e.id < 0) {
            D.esc[j] = 1;
            // reverse.setdefault((ESCAPE, d), j) over full-base escape slots
            if (e.b == D.esc_base && D.esc_slot[e.d] == 0xFFFF) D.esc_slot[e.d] = (uint16_t)j;
        } else {
            D.sym[j] = ret_sym[e.id];
            D.slot_by_digit[D.id_off[e.id] + e.d] = (uint16_t)j;
            // pad_symbol: strictly largest base, lowest slot on ties
            if (e.b > best_b) {
                best_b = e.b;
                D.pad_id = e.id;
            }
        }
    }
    D.has_pad = D.pad_id >= 0;
    D.ret_sym = ret_sym;
    D.map.init((size_t)nret);
    for (int32_t i = 0; i < nret; i++) D.map.put(ret_sym[i], i);
    D.payload_words = payload_words;
    return true;
}

// ----------------------------------------------------------------------------
// Per-row dtANS encode (codec.py:296-368) and the warp interleave
// (container.py:254-317).

struct Pos {
    uint32_t base;
    int32_t id;        // retained id, or -1 = escape
    uint64_t payload;  // escaped symbol value
};

struct Lane {
    int64_t nseg = 0;
    size_t word_off = 0, nwords = 0;   // into the slice word scratch
    size_t trace_off = 0;              // into payload/flags scratch
};

struct SliceScratch {
    std::vector<Pos> pos;
    std::vector<uint16_t> slots;
    std::vector<uint8_t> flags;  // 2 bits per segment: bit c = load at check c
    std::vector<uint32_t> words;
    std::vector<uint8_t> payload;  // per segment payload words (<= 12)
    std::vector<uint8_t> lflags;
};

static inline void pack3(const uint16_t *s, uint32_t w[3])
{
    // pack (codec.py:165-180): slot 0 least significant; w[0] most significant
    const unsigned __int128 n =
        (unsigned __int128)s[0] | ((unsigned __int128)s[1] << 12) |
        ((unsigned __int128)s[2] << 24) | ((unsigned __int128)s[3] << 36) |
        ((unsigned __int128)s[4] << 48) | ((unsigned __int128)s[5] << 60) |
        ((unsigned __int128)s[6] << 72) | ((unsigned __int128)s[7] << 84);
    w[2] = (uint32_t)n;
    w[1] = (uint32_t)(n >> 32);
    w[0] = (uint32_t)(n >> 64);
}

struct Encoder {
    const dtans_csr_view *m;
    const Domain *dom[2];
    int32_t prec;

    // Encode one row into sc.words (appended); returns false on CodingError.
    bool encode_row(int64_t row, SliceScratch &sc, Lane &lane) const
    {
        const int64_t lo = m->row_start[row], hi = m->row_start[row + 1];
        const int64_t n = 2 * (hi - lo);
        lane.nseg = (n + kL - 1) / kL;
        lane.word_off = sc.words.size();
        lane.trace_off = sc.payload.size();
        lane.nwords = 0;
        if (n == 0) return true;
        const int64_t nseg = lane.nseg;
        const int64_t P = nseg * kL;
        sc.pos.resize((size_t)P);
        sc.slots.resize((size_t)P);
        const int64_t *col = m->col_idx;
        for (int64_t t = 0; t < P; t++) {
            const int d = (int)(t & 1);
            const Domain &D = *dom[d];
            Pos &p = sc.pos[t];
            uint64_t sym;
            bool pad = t >= n;
            if (!pad) {
                const int64_t q = lo + (t >> 1);
                if (d == 0) {
                    sym = (uint64_t)(q == lo ? col[q] : col[q] - col[q - 1]);
                } else if (prec == 8) {
                    sym = ((const uint64_t *)m->values)[q];
                } else {
                    sym = ((const uint32_t *)m->values)[q];
                }
            } else {
                sym = 0;
            }
            int32_t id;
            if (pad) {
                id = D.has_pad ? D.pad_id : -1;  // escape-only table pads with payload 0
            } else {
                id = D.map.get(sym);
            }
            if (id >= 0) {
                p.base = D.id_base[id];
                p.id = id;
                p.payload = 0;
            } else {
                if (D.esc_base == 0) return false;
                p.base = (uint32_t)D.esc_base;
                p.id = -1;
                p.payload = sym;
            }
        }
        // base pass (codec.py:278-293): flags from the bases alone
        sc.flags.resize((size_t)nseg);
        {
            uint64_t r = 1;
            for (int64_t j = 0; j + 1 < nseg; j++) {
                uint8_t f = 0;
                for (int c = 0; c < kF; c++) {
                    for (int k = 4 * c; k < 4 * c + 4; k++) r *= sc.pos[j * kL + k].base;
                    if (r >= (1ull << 32)) {
                        r >>= 32;
                    } else {
                        f |= (uint8_t)(1u << c);
                    }
                }
                sc.flags[j] = f;
            }
        }
        auto slot_for = [&](int64_t t, uint64_t digit) -> uint16_t {
            const Pos &p = sc.pos[t];
            const Domain &D = *dom[t & 1];
            if (p.id < 0) return D.esc_slot[digit];
            return D.slot_by_digit[D.id_off[p.id] + digit];
        };
        // digit pass, backward (codec.py:326-365)
        const int64_t last = nseg - 1;
        for (int k = 0; k < kL; k++) sc.slots[last * kL + k] = slot_for(last * kL + k, 0);
        uint64_t d = 0;
        for (int64_t j = nseg - 2; j >= 0; j--) {
            uint32_t wn[3];
            pack3(&sc.slots[(j + 1) * kL], wn);
            for (int c = kF - 1; c >= 0; c--) {
                if (!(sc.flags[j] & (1u << c))) d = (d << 32) | wn[c];
                for (int k = 4 * c + 3; k >= 4 * c; k--) {
                    const int64_t t = j * kL + k;
                    const uint64_t b = sc.pos[t].base;
                    sc.slots[t] = slot_for(t, d % b);
                    d /= b;
                }
            }
        }
        if (d != 0) return false;  // codec.py:364 (cannot happen for valid tables)
        // forward emission in decoder consumption order
        uint32_t w[3];
        pack3(&sc.slots[0], w);
        sc.words.push_back(w[0]);
        sc.words.push_back(w[1]);
        sc.words.push_back(w[2]);
        for (int64_t j = 0; j < nseg; j++) {
            uint8_t pw = 0;
            for (int k = 0; k < kL; k++) {
                const Pos &p = sc.pos[j * kL + k];
                if (p.id >= 0) continue;
                const int nw = dom[k & 1]->payload_words;
                for (int i = 0; i < nw; i++) sc.words.push_back((uint32_t)(p.payload >> (32 * i)));
                pw = (uint8_t)(pw + nw);
            }
            sc.payload.push_back(pw);
            sc.lflags.push_back(j + 1 < nseg ? sc.flags[j] : 0);
            if (j + 1 < nseg) {
                uint32_t wn[3];
                pack3(&sc.slots[(j + 1) * kL], wn);
                if (sc.flags[j] & 1u) sc.words.push_back(wn[0]);
                if (sc.flags[j] & 2u) sc.words.push_back(wn[1]);
                sc.words.push_back(wn[2]);
            }
        }
        lane.nwords = sc.words.size() - lane.word_off;
        return true;
    }

    // Encode slice s and append its interleaved words to out.
    bool encode_slice(int64_t s, SliceScratch &sc, std::vector<uint32_t> &out) const
    {
        const int64_t row0 = s * kSlice;
        const int nl = (int)std::min<int64_t>(kSlice, m->rows - row0);
        Lane lanes[kSlice];
        sc.words.clear();
        sc.payload.clear();
        sc.lflags.clear();
        int64_t max_nseg = 0;
        for (int i = 0; i < nl; i++) {
            if (!encode_row(row0 + i, sc, lanes[i])) return false;
            max_nseg = std::max(max_nseg, lanes[i].nseg);
        }
        size_t cur[kSlice];
        for (int i = 0; i < nl; i++) cur[i] = lanes[i].word_off;
        const uint32_t *W = sc.words.data();
        // init events (container.py:263-264)
        for (int c = 0; c < kO; c++)
            for (int i = 0; i < nl; i++)
                if (lanes[i].nseg > 0) out.push_back(W[cur[i]++]);
        for (int64_t j = 0; j < max_nseg; j++) {
            // payload event
            for (int i = 0; i < nl; i++) {
                if (j >= lanes[i].nseg) continue;
                const uint8_t cnt = sc.payload[lanes[i].trace_off + j];
                for (uint8_t q = 0; q < cnt; q++) out.push_back(W[cur[i]++]);
            }
            // check events c = 0, 1 then the unconditional load
            for (int c = 0; c < kF; c++)
                for (int i = 0; i < nl; i++)
                    if (j + 1 < lanes[i].nseg && (sc.lflags[lanes[i].trace_off + j] & (1u << c)))
                        out.push_back(W[cur[i]++]);
            for (int i = 0; i < nl; i++)
                if (j + 1 < lanes[i].nseg) out.push_back(W[cur[i]++]);
        }
        for (int i = 0; i < nl; i++)
            if (cur[i] != lanes[i].word_off + lanes[i].nwords) return false;
        return true;
    }
};

static int hw_threads(int32_t req)
{
    int t = req > 0 ? req : (int)std::thread::hardware_concurrency();
    return std::max(1, std::min(t, 256));
}

template <class F>
static void parallel_for(int nthreads, int64_t n, F fn)
{
    // fn(chunk_index, lo, hi) over contiguous chunks
    if (nthreads <= 1 || n < 2) {
        fn(0, 0, n);
        return;
    }
    std::vector<std::thread> th;
    const int64_t chunk = (n + nthreads - 1) / nthreads;
    int ci = 0;
    for (int64_t lo = 0; lo < n; lo += chunk, ci++) {
        const int64_t hi = std::min(n, lo + chunk);
        th.emplace_back(fn, ci, lo, hi);
    }
    for (auto &t : th) t.join();
}

}  // namespace

int prepare_tables(const Dist &ddist, const Dist &vdist, int prec, const dtans_encode_opts *opts,
                   uint8_t *tables, Domain &Dd, Domain &Dv)
{
    const int32_t K = 1 << opts->k_log2, M = 1 << opts->m_log2;
    const uint64_t vsent = prec == 8 ? ~0ull : 0xFFFFFFFFull;
    auto quant = [&](const Dist &d, uint64_t sentinel, int raw, Quant &q) -> bool {
        std::vector<char> never(d.sym.size(), 0);
        auto it = std::lower_bound(d.sym.begin(), d.sym.end(), sentinel);
        if (it != d.sym.end() && *it == sentinel) never[it - d.sym.begin()] = 1;
        Quantizer qz(d.cnt, never, K, M, raw);
        return qz.run(q);
    };
    Quant qd, qv;
    if (!quant(ddist, kDeltaSentinel, 32, qd) || !quant(vdist, vsent, 8 * prec, qv))
        return fail(DTANS_E_PARAM, "no feasible quantization for these parameters");
    if (!build_domain(ddist, qd, opts->perm_delta, K, 1, Dd) ||
        !build_domain(vdist, qv, opts->perm_value, K, prec / 4, Dv))
        return fail(DTANS_E_PARAM, "permutation must be a bijection on slots");

    // tables block (container.py:612-625)
    const int rec = prec == 8 ? 16 : 12;
    for (int32_t j = 0; j < K; j++) {
        uint8_t *r = tables + (size_t)j * rec;
        const uint64_t vs = Dv.esc[j] ? vsent : Dv.sym[j];
        const uint32_t ds = Dd.esc[j] ? (uint32_t)kDeltaSentinel : (uint32_t)Dd.sym[j];
        if (prec == 8) {
            memcpy(r, &vs, 8);
            memcpy(r + 8, &ds, 4);
            r += 12;
        } else {
            const uint32_t v32 = (uint32_t)vs;
            memcpy(r, &v32, 4);
            memcpy(r + 4, &ds, 4);
            r += 8;
        }
        r[0] = Dd.dig[j];
        r[1] = (uint8_t)(Dd.base[j] - 1);
        r[2] = Dv.dig[j];
        r[3] = (uint8_t)(Dv.base[j] - 1);
    }
    return DTANS_OK;
}

}  // namespace dtans

using namespace dtans;

extern "C" const char *dtans_last_error(void) { return g_last_error.c_str(); }
extern "C" int dtans_abi_version(void) { return 1; }

extern "C" int dtans_quantize(int64_t n, const uint64_t *symbols, const int64_t *counts,
                              int32_t k, int32_t m, int32_t raw_width_bits, int64_t n_never,
                              const uint64_t *never_retain, int32_t *mult, int32_t *esc_mult,
                              int32_t *esc_slots)
{
    if (k < 2) return fail(DTANS_E_PARAM, "k must be >= 2");
    if (m < 1 || m > k) return fail(DTANS_E_PARAM, "need 1 <= m <= k");
    std::vector<int64_t> cnt(counts, counts + n);
    std::vector<char> never(n, 0);
    for (int64_t i = 0; i < n; i++) {
        if (cnt[i] < 1) return fail(DTANS_E_PARAM, "counts must be integers >= 1");
        for (int64_t j = 0; j < n_never; j++)
            if (symbols[i] == never_retain[j]) never[i] = 1;
    }
    Quantizer qz(cnt, never, k, m, raw_width_bits);
    Quant q;
    if (!qz.run(q)) return fail(DTANS_E_PARAM, "no feasible quantization for these parameters");
    for (int64_t i = 0; i < n; i++) mult[i] = q.mult[i];
    *esc_mult = q.esc_mult;
    *esc_slots = q.esc_slots;
    return DTANS_OK;
}

extern "C" void dtans_encoded_free(dtans_encoded *e)
{
    if (!e) return;
    free(e->tables);
    free(e->row_symbols);
    free(e->directory);
    free(e->stream);
    e->tables = nullptr;
    e->row_symbols = nullptr;
    e->directory = nullptr;
    e->stream = nullptr;
}

extern "C" int dtans_encode(const dtans_csr_view *m, const dtans_encode_opts *opts,
                            dtans_encoded *out)
{
    try {
        if (!m || !opts || !out) return fail(DTANS_E_PARAM, "null argument");
        memset(out, 0, sizeof(*out));
        const int prec = m->precision;
        if (prec != 4 && prec != 8) return fail(DTANS_E_PARAM, "precision must be 4 or 8 bytes");
        if (opts->k_log2 != kKLog2) return fail(DTANS_E_PARAM, "this build implements k = 4096");
        if (opts->m_log2 < 1 || opts->m_log2 > 8)
            return fail(DTANS_E_PARAM, "slot records store base - 1 in one byte; m <= 256");
        const int32_t K = 1 << opts->k_log2;
        if (m->rows < 0 || m->cols < 0) return fail(DTANS_E_PARAM, "negative dimensions");
        if (m->cols > (int64_t)1 << 32 || m->rows > (int64_t)1 << 32)
            return fail(DTANS_E_PARAM, "indices must fit 32 bits");
        const int64_t rows = m->rows, nnz = m->nnz;
        const int64_t *rs = m->row_start;
        // CsrMatrix.validate (sparse.py:76-91)
        if (rs[0] != 0 || rs[rows] != nnz) return fail(DTANS_E_PARAM, "row_start must span [0, nnz]");
        for (int64_t i = 0; i < rows; i++)
            if (rs[i + 1] < rs[i]) return fail(DTANS_E_PARAM, "row_start must be nondecreasing");
        const int T = hw_threads(opts->threads);
        const int64_t nslices = (rows + kSlice - 1) / kSlice;

        // Chunks of whole rows, balanced by nnz, for the statistics pass.
        std::vector<int64_t> row_cut(T + 1, rows);
        row_cut[0] = 0;
        for (int t = 1; t < T; t++) {
            const int64_t target = nnz / T * t;
            row_cut[t] = std::upper_bound(rs, rs + rows + 1, target) - rs - 1;
            if (row_cut[t] < row_cut[t - 1]) row_cut[t] = row_cut[t - 1];
        }
        std::vector<std::vector<uint64_t>> dsy(T), vsy(T);
        std::vector<std::vector<int64_t>> dct(T), vct(T);
        std::atomic<int> bad{0};
        {
            std::vector<std::thread> th;
            for (int t = 0; t < T; t++) {
                th.emplace_back([&, t]() {
                    const int64_t r0 = row_cut[t], r1 = row_cut[t + 1];
                    const int64_t p0 = rs[r0], p1 = rs[r1];
                    std::vector<uint64_t> buf((size_t)(p1 - p0));
                    const int64_t *col = m->col_idx;
                    for (int64_t r = r0; r < r1; r++) {
                        for (int64_t q = rs[r]; q < rs[r + 1]; q++) {
                            const int64_t c = col[q];
                            if (c < 0 || c >= m->cols) { bad = 1; return; }
                            if (q > rs[r] && c <= col[q - 1]) { bad = 2; return; }
                            buf[q - p0] = (uint64_t)(q == rs[r] ? c : c - col[q - 1]);
                        }
                    }
                    std::sort(buf.begin(), buf.end());
                    rle_sorted(buf.data(), buf.size(), dsy[t], dct[t]);
                    if (prec == 8) {
                        const uint64_t *v = (const uint64_t *)m->values;
                        std::copy(v + p0, v + p1, buf.begin());
                    } else {
                        const uint32_t *v = (const uint32_t *)m->values;
                        for (int64_t q = p0; q < p1; q++) buf[q - p0] = v[q];
                    }
                    std::sort(buf.begin(), buf.end());
                    rle_sorted(buf.data(), buf.size(), vsy[t], vct[t]);
                });
            }
            for (auto &x : th) x.join();
        }
        if (bad == 1) return fail(DTANS_E_PARAM, "column index out of range");
        if (bad == 2) return fail(DTANS_E_PARAM, "columns must be strictly ascending per row");
        Dist ddist = merge_runs(dsy, dct);
        Dist vdist = merge_runs(vsy, vct);

        Domain Dd, Dv;
        const int rec = prec == 8 ? 16 : 12;
        out->tables = (uint8_t *)malloc((size_t)K * rec);
        out->row_symbols = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)std::max<int64_t>(rows, 1));
        out->directory = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(nslices + 1));
        if (!out->tables || !out->row_symbols || !out->directory) {
            dtans_encoded_free(out);
            return fail(DTANS_E_NOMEM, "host allocation failed");
        }
        {
            const int rc = prepare_tables(ddist, vdist, prec, opts, out->tables, Dd, Dv);
            if (rc) {
                dtans_encoded_free(out);
                return rc;
            }
        }
        for (int64_t i = 0; i < rows; i++) out->row_symbols[i] = (uint32_t)(2 * (rs[i + 1] - rs[i]));

        // per-slice encode + interleave, chunks of whole slices balanced by nnz
        Encoder enc;
        enc.m = m;
        enc.dom[0] = &Dd;
        enc.dom[1] = &Dv;
        enc.prec = prec;
        const int TS = (int)std::max<int64_t>(1, std::min<int64_t>(T * 4, nslices));
        std::vector<int64_t> sl_cut(TS + 1, nslices);
        sl_cut[0] = 0;
        for (int t = 1; t < TS; t++) {
            const int64_t target = nnz / TS * t;
            int64_t r = std::upper_bound(rs, rs + rows + 1, target) - rs - 1;
            sl_cut[t] = std::max(sl_cut[t - 1], std::min(nslices, r / kSlice));
        }
        std::vector<std::vector<uint32_t>> chunk_words(TS);
        std::vector<int64_t> slice_words((size_t)nslices, 0);
        std::atomic<int> next{0};
        std::atomic<int> enc_bad{0};
        {
            std::vector<std::thread> th;
            for (int t = 0; t < std::min(T, TS); t++) {
                th.emplace_back([&]() {
                    SliceScratch sc;
                    for (;;) {
                        const int ci = next.fetch_add(1);
                        if (ci >= TS) break;
                        auto &ow = chunk_words[ci];
                        for (int64_t s = sl_cut[ci]; s < sl_cut[ci + 1]; s++) {
                            const size_t before = ow.size();
                            if (!enc.encode_slice(s, sc, ow)) { enc_bad = 1; return; }
                            slice_words[s] = (int64_t)(ow.size() - before);
                        }
                    }
                });
            }
            for (auto &x : th) x.join();
        }
        if (enc_bad) {
            dtans_encoded_free(out);
            return fail(DTANS_E_CODING, "symbol not retained and its table has no escape entry");
        }
        out->directory[0] = 0;
        for (int64_t s = 0; s < nslices; s++) out->directory[s + 1] = out->directory[s] + slice_words[s];
        const int64_t nwords = (int64_t)out->directory[nslices];
        out->stream = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)std::max<int64_t>(nwords, 1));
        if (!out->stream) {
            dtans_encoded_free(out);
            return fail(DTANS_E_NOMEM, "host allocation failed");
        }
        parallel_for(T, TS, [&](int, int64_t lo, int64_t hi) {
            for (int64_t ci = lo; ci < hi; ci++) {
                if (sl_cut[ci] >= sl_cut[ci + 1]) continue;
                const auto &ow = chunk_words[ci];
                if (!ow.empty())
                    memcpy(out->stream + out->directory[sl_cut[ci]], ow.data(), ow.size() * 4);
            }
        });
        out->rows = rows;
        out->cols = m->cols;
        out->nnz = nnz;
        out->nslices = nslices;
        out->nwords = nwords;
        out->precision = prec;
        out->rec_size = rec;
        return DTANS_OK;
    } catch (const std::bad_alloc &) {
        dtans_encoded_free(out);
        return fail(DTANS_E_NOMEM, "host allocation failed");
    }
}
