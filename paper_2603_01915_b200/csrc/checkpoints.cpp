// Long-slice checkpoint index (host, C++17, multithreaded).
//
// A slice whose longest row needs more than `seg_threshold` segments is one
// serial chain per lane: the reference decoder (container.py:370-521) walks
// it segment by segment and so would one warp.  At upload we walk such slices
// once on the host, replaying the same lockstep consumption (init events,
// payload events, two conditional checks and one unconditional load per
// segment; container.py:254-280, 406-497), and record every `chunk` segments
// the state each still-active lane needs to resume: its three words, the
// mixed-radix pair (d, r) and its running column, plus the slice cursor.
// The SpMV then decodes the segment ranges between checkpoints as
// independent warp tasks and combines the per-task partial sums in order.
// The index is auxiliary: the container bytes are unchanged.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <thread>
#include <vector>

#include "checkpoints.h"
#include "common.h"

namespace dtans {

namespace {

struct HostTables {
    uint8_t esc[2][kK];
    uint8_t dig[2][kK];
    uint8_t bm1[2][kK];
    uint8_t pw[2];  // payload words per escape: delta 1, value prec/4
};

void parse_tables(const uint8_t *recs, int precision, HostTables &t)
{
    const int rec = precision == 8 ? 16 : 12;
    const uint64_t vsent = precision == 8 ? ~0ull : 0xFFFFFFFFull;
    for (int j = 0; j < kK; j++) {
        const uint8_t *r = recs + (size_t)j * rec;
        uint64_t vs = 0;
        uint32_t ds = 0;
        if (precision == 8) {
            memcpy(&vs, r, 8);
            memcpy(&ds, r + 8, 4);
            r += 12;
        } else {
            uint32_t v32;
            memcpy(&v32, r, 4);
            vs = v32;
            memcpy(&ds, r + 4, 4);
            r += 8;
        }
        t.esc[0][j] = ds == (uint32_t)kDeltaSentinel;
        t.esc[1][j] = vs == vsent;
        t.dig[0][j] = r[0];
        t.bm1[0][j] = r[1];
        t.dig[1][j] = r[2];
        t.bm1[1][j] = r[3];
    }
    t.pw[0] = 1;
    t.pw[1] = (uint8_t)(precision / 4);
}

// Walk one slice; append checkpoints for segments chunk, 2*chunk, ...
// Returns false on a corrupt slice (reads past the stream or consumption
// mismatch).  Column deltas need the symbols, so escapes' payloads and the
// delta dictionary are read like the device does.
bool walk_slice(const dtans_container_view *c, const HostTables &T, const uint32_t *dsym_tab, int64_t s,
                int chunk, std::vector<uint32_t> &pool, std::vector<LongTask> &tasks, std::vector<SoloTask> &solo,
                uint32_t part_base)
{
    const int64_t row0 = s * kSlice;
    const int nl = (int)std::min<int64_t>(kSlice, c->rows - row0);
    const uint64_t lo = c->directory[s], hi = c->directory[s + 1];
    const uint32_t *st = c->stream + lo;
    const uint64_t nw = hi - lo;
    uint32_t n[kSlice] = {0}, nseg[kSlice] = {0};
    uint32_t w0[kSlice] = {0}, w1[kSlice] = {0}, w2[kSlice] = {0}, d[kSlice] = {0}, r[kSlice], col[kSlice] = {0};
    uint32_t max_nseg = 0;
    for (int i = 0; i < kSlice; i++) r[i] = 1;
    for (int i = 0; i < nl; i++) {
        n[i] = c->row_symbols[row0 + i];
        nseg[i] = (n[i] + 7) / 8;
        max_nseg = std::max(max_nseg, nseg[i]);
    }
    uint64_t cur = 0;
    auto fetch = [&](uint32_t &dst) -> bool {
        if (cur >= nw) return false;
        dst = st[cur++];
        return true;
    };
    for (int i = 0; i < nl; i++)
        if (nseg[i] && !fetch(w0[i])) return false;
    for (int i = 0; i < nl; i++)
        if (nseg[i] && !fetch(w1[i])) return false;
    for (int i = 0; i < nl; i++)
        if (nseg[i] && !fetch(w2[i])) return false;
    const uint32_t ntasks = (max_nseg + chunk - 1) / chunk;
    uint32_t k = 0;
    const size_t first_task = tasks.size(), first_solo = solo.size();
    for (uint32_t j = 0; j < max_nseg; j++) {
        uint32_t amask = 0;
        if (j % chunk == 0 && j)
            for (int i = 0; i < nl; i++)
                if (nseg[i] > j) amask |= 1u << i;
        if (j % chunk == 0 && j && __builtin_popcount(amask) == 1) {
            // one lane left: its remaining words are consecutive (solo task)
            const int i = __builtin_ctz(amask);
            SoloTask t;
            t.slice = (uint32_t)s;
            t.lane = (uint32_t)i;
            t.j0 = j;
            t.j1 = std::min<uint32_t>(j + chunk, max_nseg);
            t.part = part_base + k;
            t.cur0 = (uint32_t)cur;
            t.cur1 = 0;
            t.ck = (uint32_t)pool.size();
            pool.push_back(w0[i]);
            pool.push_back(w1[i]);
            pool.push_back(w2[i]);
            pool.push_back(d[i]);
            pool.push_back(r[i]);
            pool.push_back(col[i]);
            solo.push_back(t);
            k++;
        } else if (j % chunk == 0) {
            // task k covers segments [j, min(j + chunk, max_nseg))
            LongTask t;
            t.slice = (uint32_t)s;
            t.j0 = j;
            t.j1 = std::min<uint32_t>(j + chunk, max_nseg);
            t.part = part_base + k;
            t.cur0 = (uint32_t)cur;
            t.ck = j == 0 ? 0xFFFFFFFFu : (uint32_t)pool.size();
            t.last = k + 1 == ntasks;
            if (j) {
                uint32_t mask = 0;
                for (int i = 0; i < nl; i++)
                    if (nseg[i] > j) mask |= 1u << i;
                pool.push_back(mask);
                for (int i = 0; i < nl; i++)
                    if (mask >> i & 1u) {
                        pool.push_back(w0[i]);
                        pool.push_back(w1[i]);
                        pool.push_back(w2[i]);
                        pool.push_back(d[i]);
                        pool.push_back(r[i]);
                        pool.push_back(col[i]);
                    }
            }
            tasks.push_back(t);
            k++;
        }
        uint32_t slot[kSlice][8];
        for (int i = 0; i < nl; i++) {
            if (j >= nseg[i]) continue;
            const unsigned __int128 num =
                ((unsigned __int128)w0[i] << 64) | ((unsigned __int128)w1[i] << 32) | (unsigned __int128)w2[i];
            for (int q = 0; q < 8; q++) slot[i][q] = (uint32_t)((num >> (12 * q)) & 0xFFFu);
        }
        // payload event: lanes in order, slots in order
        for (int i = 0; i < nl; i++) {
            if (j >= nseg[i]) continue;
            for (int q = 0; q < 8; q++) {
                const int dom = q & 1;
                const uint32_t sl = slot[i][q];
                uint32_t first = 0;
                if (T.esc[dom][sl]) {
                    for (int p = 0; p < T.pw[dom]; p++) {
                        uint32_t wd;
                        if (!fetch(wd)) return false;
                        if (p == 0) first = wd;
                    }
                }
                if (dom == 0 && 8 * j + q < n[i]) col[i] += T.esc[0][sl] ? first : dsym_tab[sl];
            }
        }
        for (int g = 0; g < 2; g++) {
            for (int i = 0; i < nl; i++) {
                if (j + 1 >= nseg[i]) continue;
                uint64_t dd = d[i], rr = r[i];
                for (int q = 4 * g; q < 4 * g + 4; q++) {
                    const int dom = q & 1;
                    const uint64_t b1 = T.bm1[dom][slot[i][q]];
                    dd = dd * b1 + dd + T.dig[dom][slot[i][q]];
                    rr = rr * b1 + rr;
                }
                uint32_t &wg = g == 0 ? w0[i] : w1[i];
                if (rr >> 32) {
                    wg = (uint32_t)dd;
                    d[i] = (uint32_t)(dd >> 32);
                    r[i] = (uint32_t)(rr >> 32);
                } else {
                    d[i] = (uint32_t)dd;
                    r[i] = (uint32_t)rr;
                    if (!fetch(wg)) return false;
                }
            }
        }
        for (int i = 0; i < nl; i++)
            if (j + 1 < nseg[i] && !fetch(w2[i])) return false;
        // the next task's start cursor
    }
    // expected cursor at each task end = the next task's start, last = nwords
    // (warp tasks precede the solo tasks of the same slice)
    std::vector<uint32_t *> ends;
    std::vector<uint32_t> starts;
    for (size_t t = first_task; t < tasks.size(); t++) {
        ends.push_back(&tasks[t].cur1);
        starts.push_back(tasks[t].cur0);
    }
    for (size_t t = first_solo; t < solo.size(); t++) {
        ends.push_back(&solo[t].cur1);
        starts.push_back(solo[t].cur0);
    }
    for (size_t q = 0; q < ends.size(); q++) *ends[q] = q + 1 < ends.size() ? starts[q + 1] : (uint32_t)nw;
    (void)ntasks;
    return cur == nw;
}

}  // namespace

int build_long_index(const dtans_container_view *c, int seg_threshold, uint64_t max_words, int chunk,
                     LongIndex &out)
{
    out = LongIndex();
    const int64_t nsl = c->nslices;
    std::vector<uint32_t> longs;
    for (int64_t s = 0; s < nsl; s++) {
        const int64_t row0 = s * kSlice, row1 = std::min<int64_t>(row0 + kSlice, c->rows);
        uint32_t mx = 0;
        for (int64_t i = row0; i < row1; i++) mx = std::max(mx, c->row_symbols[i]);
        const uint64_t words = ((c->directory[s + 1] + 3) & ~3ull) - (c->directory[s] & ~3ull);
        if ((mx + 7) / 8 > (uint32_t)seg_threshold || words > max_words) longs.push_back((uint32_t)s);
    }
    if (longs.empty()) return DTANS_OK;
    HostTables T;
    parse_tables(c->tables, c->precision, T);
    // delta dictionary by slot (escape slots are never read through it)
    std::vector<uint32_t> dsym(kK, 0);
    {
        const int rec = c->precision == 8 ? 16 : 12;
        for (int j = 0; j < kK; j++) memcpy(&dsym[j], c->tables + (size_t)j * rec + (c->precision == 8 ? 8 : 4), 4);
    }
    // partial-slot bases in slice order
    std::vector<uint32_t> base(longs.size() + 1, 0);
    for (size_t i = 0; i < longs.size(); i++) {
        const int64_t s = longs[i];
        const int64_t row0 = s * kSlice, row1 = std::min<int64_t>(row0 + kSlice, c->rows);
        uint32_t mx = 0;
        for (int64_t r = row0; r < row1; r++) mx = std::max(mx, c->row_symbols[r]);
        base[i + 1] = base[i] + ((mx + 7) / 8 + chunk - 1) / chunk;
    }
    const int nt = std::max(1, std::min<int>((int)std::thread::hardware_concurrency(), (int)longs.size()));
    std::vector<std::vector<uint32_t>> pools(nt);
    std::vector<std::vector<LongTask>> tasks(nt);
    std::vector<std::vector<SoloTask>> solos(nt);
    std::atomic<size_t> next{0};
    std::atomic<int> bad{0};
    std::vector<std::thread> th;
    for (int t = 0; t < nt; t++)
        th.emplace_back([&, t]() {
            for (;;) {
                const size_t i = next.fetch_add(1);
                if (i >= longs.size()) break;
                if (!walk_slice(c, T, dsym.data(), longs[i], chunk, pools[t], tasks[t], solos[t], base[i])) bad = 1;
            }
        });
    for (auto &x : th) x.join();
    if (bad) return fail(DTANS_E_CORRUPT, "long slice consumed an unexpected number of words");
    for (int t = 0; t < nt; t++) {
        const uint32_t off = (uint32_t)out.pool.size();
        for (auto tk : tasks[t]) {
            if (tk.ck != 0xFFFFFFFFu) tk.ck += off;
            out.tasks.push_back(tk);
        }
        for (auto tk : solos[t]) {
            tk.ck += off;
            out.solo.push_back(tk);
        }
        out.pool.insert(out.pool.end(), pools[t].begin(), pools[t].end());
    }
    // longest tasks first (LPT) so the tail of the task kernel is short
    std::stable_sort(out.tasks.begin(), out.tasks.end(),
                     [](const LongTask &a, const LongTask &b) { return a.j1 - a.j0 > b.j1 - b.j0; });
    std::stable_sort(out.solo.begin(), out.solo.end(),
                     [](const SoloTask &a, const SoloTask &b) { return a.j1 - a.j0 > b.j1 - b.j0; });
    // finalize order: slices with <= 32 partials first (warp per slice), then
    // the rest (CTA per slice)
    for (int pass = 0; pass < 2; pass++)
        for (size_t i = 0; i < longs.size(); i++) {
            const uint32_t np = base[i + 1] - base[i];
            if ((np <= 32) == (pass == 0)) out.slices.push_back(LongSlice{longs[i], base[i], np, 0});
        }
    out.nparts = base.back();
    if (out.pool.empty()) out.pool.push_back(0);
    return DTANS_OK;
}

}  // namespace dtans
