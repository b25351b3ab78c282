// Fused dtANS decode + SpMV for sm_100a.
//
// Mapping.  One warp decodes one 32-row slice, lane i = row 32s+i: exactly
// the lockstep the container's word order was interleaved for
// (container.py:211-335).  Per lane the decoder runs the reference's
// per-segment loop (container.py:370-521, codec.py:384-453):
//   unpack 3 words -> 8 slots, 8 slot-table lookups (shared memory),
//   escape payload event (warp exclusive scan), 2 mixed-radix checks
//   (extract from the state, or load: ballot + popc), 1 unconditional load.
// The symbols never leave registers: column deltas are prefix-summed,
// x[col] is gathered, acc = fl(acc + fl(v * x)) runs left to right per row
// from +0.0 (container.py:534-551) with __dmul_rn/__dadd_rn, so the result
// is bitwise the reference's.
//
// Memory.  Each warp owns a ring of kRing shared-memory buffers; lane 0
// stages the word range [directory[s], directory[s+1]) of the slice it will
// decode kRing slices later with one cp.async.bulk (TMA bulk copy, 16-byte
// aligned window) completing on an mbarrier.  The decoder then reads stream
// words from shared memory.  Slices larger than a buffer are read straight
// from global memory (same code, generic pointer).  Slot tables are compact
// u32 entries {digit:8, base-1:8, id:16} per domain (16 KB each) plus
// dictionaries of the retained symbols, so a CTA needs ~33 KB of tables.
//
// Mixed-radix state.  At every segment start d < r < 2^32 (r is divided by
// 2^32 whenever it reaches 2^32), so the resting state is two u32.  A group
// of 4 digits folds into one product in 32-bit arithmetic with the
// decremented radix Bm1 = b0 b1 b2 b3 - 1 <= 2^32 - 1 (codec.py:127-137):
//   d' = d*Bm1 + d + D,  r' = r*Bm1 + r       (64-bit, < 2^64)
// and the check is r' >= 2^32: extract w = lo32(d'), d = hi32(d'),
// r = hi32(r'); else load (d', r' already fit 32 bits).
#pragma once
#include <cstdint>

#include "checkpoints.h"

namespace dtans {
namespace dev {

constexpr int kSliceRows = 32;
constexpr int kSlots = 4096;
constexpr int kMaxWarps = 32;  // per CTA (1024 threads); smem layout is sized for this
constexpr int kRing = 3;

template <typename V> struct ValueTraits;
template <> struct ValueTraits<double> {
    using Bits = unsigned long long;
    static constexpr int kPayloadWords = 2;
    __device__ static inline double from_bits(Bits b) { return __longlong_as_double((long long)b); }
    __device__ static inline double mul(double a, double b) { return __dmul_rn(a, b); }
    __device__ static inline double add(double a, double b) { return __dadd_rn(a, b); }
};
template <> struct ValueTraits<float> {
    using Bits = uint32_t;
    static constexpr int kPayloadWords = 1;
    __device__ static inline float from_bits(Bits b) { return __uint_as_float(b); }
    __device__ static inline float mul(float a, float b) { return __fmul_rn(a, b); }
    __device__ static inline float add(float a, float b) { return __fadd_rn(a, b); }
};

struct KernelArgs {
    const uint32_t *tables;       // [dtab 4096][vtab 4096][ddict][vdict] (global copy)
    int32_t table_bytes;          // bytes to copy into shared memory (multiple of 16)
    int32_t off_ddict, off_vdict; // byte offsets inside the table block
    uint32_t desc_min, vesc_min;  // entry >= this  <=>  escape (id == n_retained)
    int32_t pads_ok;              // both domains retain a pad symbol
    int32_t off_bars, off_meta, off_bufs;  // shared-memory layout
    int32_t bufw;                 // words per stream buffer
    const uint32_t *row_symbols;  // rows
    const uint64_t *directory;    // nslices + 1
    const uint32_t *stream;       // nwords (+ 64 B padding)
    int64_t rows, cols, nslices, nwords;
    const void *x;
    const void *y;                // may be null (y' = A x)
    void *out;
    const int64_t *row_start;     // decode kernel only
    int64_t *dec_cols;            // decode kernel only
    void *dec_vals;               // decode kernel only
    unsigned int *err;            // bit 0: consumption mismatch, bit 1: column OOB
    // long slices (checkpoint index, checkpoints.cpp)
    uint32_t long_seg;            // slices with more segments go to the task kernel
    uint32_t long_words;          // ... and slices with more stream words
    uint32_t ntasks, nlong, nsolo;
    uint32_t nlong_small, nlong_small_blocks;  // finalize: slices with <= 32 partials come first
    int32_t single_direct;                      // single-task slices write y' in the task kernel
    const LongTask *tasks;
    const SoloTask *solo;
    const uint32_t *ck_pool;
    const LongSlice *longs;
    void *partials;               // V[nparts][32]
    const uint32_t *row_map;      // optional: y/out index of encoded row i (row-reordered P*A)
    // work distribution
    int32_t dynamic;              // 1: atomic ticket counter instead of a static stride
    uint32_t slice_lo, slice_hi;  // static order: slices [slice_lo, slice_hi) of this launch
    uint32_t *work_counter;       // zeroed before every dynamic launch
    const uint32_t *slice_order;  // optional: ticket -> slice (longest first)
};

__device__ __forceinline__ uint32_t lanemask_lt()
{
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void fence_proxy_async()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void fence_mbar_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ uint32_t lds32(uint32_t addr)
{
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ unsigned long long lds64(uint32_t addr)
{
    unsigned long long v;
    asm("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(addr));
    return v;
}

// Stream words that change between slices (TMA-written): volatile so they
// are never hoisted across the mbarrier wait.
__device__ __forceinline__ uint32_t lds32_v(uint32_t addr)
{
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

template <typename Bits> __device__ __forceinline__ Bits lds_bits(uint32_t addr);
template <> __device__ __forceinline__ unsigned long long lds_bits<unsigned long long>(uint32_t addr)
{
    return lds64(addr);
}
template <> __device__ __forceinline__ uint32_t lds_bits<uint32_t>(uint32_t addr) { return lds32(addr); }

// Word sources for one slice, addressed by the position relative to
// directory[s] (32-bit): the staged shared-memory window or global memory.
// Reads are not clamped: a segment consumes at most kSegMaxWords words, the
// decoder stops as soon as its cursor passes the slice end (then reports
// CorruptStream), and both the shared ring and the device stream carry at
// least kOverrunWords of slack, so a corrupt container can never read
// outside the allocations.
constexpr uint32_t kSegMaxWords = 32u * 15u;  // payload 12 + 2 checks + 1 uncond per lane
constexpr uint32_t kOverrunWords = 3u * 32u + kSegMaxWords + 64u;
constexpr uint32_t kStreamPadWords = kOverrunWords;  // device stream padding
struct SmemSrc {
    uint32_t addr;  // shared address of word directory[s]
    __device__ __forceinline__ uint32_t operator()(uint32_t rel) const { return lds32_v(addr + rel * 4u); }
    __device__ __forceinline__ void advance(uint32_t, int) {}
};
struct GmemSrc {
    const uint32_t *p;  // &stream[directory[s]]
    __device__ __forceinline__ uint32_t operator()(uint32_t rel) const { return __ldg(p + rel); }
    __device__ __forceinline__ void advance(uint32_t, int) {}
};


// Per-buffer slice record written by the stager: the slice's word offset
// inside the 16-byte aligned staged window (bit 31: not staged, read from
// global memory instead) and its word count.
struct SliceMeta {
    uint32_t off;     // words from the window start to directory[s]; bit 31 = global
    uint32_t nwords;  // directory[s+1] - directory[s]
    uint32_t slice;   // slice id (kNoSlice: the warp's work is exhausted)
    uint32_t pad;
};
constexpr uint32_t kNoSlice = 0xFFFFFFFFu;
constexpr uint32_t kGlobalSlice = 0x80000000u;

// Stage a slice (directory entries lo, hi prefetched) into a ring buffer
// (lane 0 only).  The previous contents were consumed by this warp's LDS
// before the __syncwarp that precedes the call (the same WAR ordering a
// CUTLASS TMA pipeline relies on), so no proxy fence is issued.
__device__ __forceinline__ void stage_slice(const KernelArgs &a, uint32_t s, uint64_t lo, uint64_t hi,
                                            uint64_t *bar, SliceMeta *meta, uint32_t *buf)
{
    if (s == kNoSlice) {
        *meta = SliceMeta{0u, 0u, kNoSlice, 0u};
        mbar_arrive(bar);
        return;
    }
    const uint64_t abase = lo & ~3ull;
    const uint32_t words = (uint32_t)(((hi + 3) & ~3ull) - abase);
    const bool staged = words > 0 && words <= (uint32_t)a.bufw;
    *meta = SliceMeta{(uint32_t)(lo - abase) | (staged ? 0u : kGlobalSlice), (uint32_t)(hi - lo), s, 0u};
    if (staged) {
        mbar_arrive_expect_tx(bar, words * 4u);
        bulk_g2s(buf, a.stream + abase, words * 4u, bar);
    } else {
        mbar_arrive(bar);
    }
}

struct Ctx {
    uint32_t dtab, vtab, ddict, vdict;  // shared addresses
    uint32_t desc_min, vesc_min;        // entry >= this <=> escape
    uint32_t cols_m1;
    uint32_t lt;                        // lanemask_lt
    bool pads_ok;
};

__device__ __forceinline__ void slot_offsets(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t so[8])
{
    // unpack (codec.py:148-162): slot k = bits [12k, 12k+12) of w0:w1:w2, as
    // byte offsets (slot * 4) into the u32 slot tables
    so[0] = (w2 << 2) & 0x3FFCu;
    so[1] = (w2 >> 10) & 0x3FFCu;
    so[2] = __funnelshift_r(w2, w1, 22) & 0x3FFCu;
    so[3] = (w1 >> 2) & 0x3FFCu;
    so[4] = (w1 >> 14) & 0x3FFCu;
    so[5] = __funnelshift_r(w1, w0, 26) & 0x3FFCu;
    so[6] = (w0 >> 6) & 0x3FFCu;
    so[7] = (w0 >> 18) & 0x3FFCu;
}

// Table entries of pair p and the dictionary symbols they point at (escape
// entries point at a dummy dictionary slot; the payload overwrites them).
template <typename Bits>
__device__ __forceinline__ void lookup_pair(const Ctx &C, uint32_t sod, uint32_t sov, uint32_t &ed, uint32_t &ev,
                                            uint32_t &ds, Bits &vs)
{
    ed = lds32(C.dtab + sod);
    ev = lds32(C.vtab + sov);
    ds = lds32(C.ddict + (ed >> 16));  // id field = byte offset into the dictionary
    vs = lds_bits<Bits>(C.vdict + (ev >> 16));
}

// Payload event (container.py:459-470): per-lane word counts, exclusive warp
// scan, words read in slot order, low word first, overwriting the symbols.
template <typename T, class Src>
__device__ __forceinline__ void payload_event(const Ctx &C, const Src &src, uint32_t &cur, const bool act,
                                              const uint32_t e[8], uint32_t ds[4], typename T::Bits vs[4],
                                              const int lane)
{
    using Bits = typename T::Bits;
    // cheap test first: escape entries are the largest entries of a table
    const uint32_t dmax = max(max(e[0], e[2]), max(e[4], e[6]));
    const uint32_t vmax = max(max(e[1], e[3]), max(e[5], e[7]));
    const bool has = act && (dmax >= C.desc_min || vmax >= C.vesc_min);
    if (!__any_sync(0xFFFFFFFFu, has)) return;
    uint32_t pc = 0;
#pragma unroll
    for (int p = 0; p < 4; p++)
        pc += (e[2 * p] >= C.desc_min ? 1u : 0u) + (e[2 * p + 1] >= C.vesc_min ? (uint32_t)T::kPayloadWords : 0u);
    if (!act) pc = 0;
    const uint32_t any = __ballot_sync(0xFFFFFFFFu, pc != 0);
    if (__all_sync(0xFFFFFFFFu, pc <= 1u)) {
        // common case (e.g. one escaped first column per row): every lane
        // reads at most one word, its rank among the escaping lanes
        const uint32_t w = src(cur + __popc(any & C.lt));
#pragma unroll
        for (int p = 0; p < 4; p++) {
            if (e[2 * p] >= C.desc_min) ds[p] = w;
            if (T::kPayloadWords == 1 && e[2 * p + 1] >= C.vesc_min) vs[p] = (Bits)w;
        }
        cur += __popc(any);
        return;
    }
    // exclusive warp scan of pc (<= 12 words: 4 bit planes), one ballot per
    // plane: independent ballots instead of a dependent 5-step shuffle chain
    const uint32_t b1 = __ballot_sync(0xFFFFFFFFu, pc & 2u);
    const uint32_t b2 = __ballot_sync(0xFFFFFFFFu, pc & 4u);
    const uint32_t b3 = __ballot_sync(0xFFFFFFFFu, pc & 8u);
    const uint32_t b0 = __ballot_sync(0xFFFFFFFFu, pc & 1u);
    const uint32_t excl = __popc(b0 & C.lt) + (__popc(b1 & C.lt) << 1) + (__popc(b2 & C.lt) << 2) +
                          (__popc(b3 & C.lt) << 3);
    const uint32_t incl = excl + pc;
    const uint32_t total = __popc(b0) + (__popc(b1) << 1) + (__popc(b2) << 2) + (__popc(b3) << 3);
    if (pc) {
        uint32_t off = cur + (incl - pc);
#pragma unroll
        for (int p = 0; p < 4; p++) {
            if (e[2 * p] >= C.desc_min) {
                ds[p] = src(off);
                off += 1;
            }
            if (e[2 * p + 1] >= C.vesc_min) {
                if (T::kPayloadWords == 2) {
                    const uint32_t lo = src(off), hi = src(off + 1);
                    vs[p] = (Bits)(((unsigned long long)hi << 32) | lo);
                } else {
                    vs[p] = (Bits)src(off);
                }
                off += T::kPayloadWords;
            }
        }
    }
    cur += total;
}

__device__ __forceinline__ uint32_t byte1(uint32_t x) { return __byte_perm(x, 0u, 0x4441u); }

// Group of 4 slots -> decremented radix Bm1 = b0 b1 b2 b3 - 1 and digit D,
// using b*x = bm1*x + x so no "+1" is needed (codec.py:127-137).
__device__ __forceinline__ void group(uint32_t m0, uint32_t m1, uint32_t m2, uint32_t m3, uint32_t &bm1,
                                      uint32_t &dg)
{
    const uint32_t q0 = byte1(m0), q1 = byte1(m1), q2 = byte1(m2), q3 = byte1(m3);
    uint32_t P = q0 + 1u;       // b0
    P = P * q1 + P;             // b0 b1
    P = P * q2 + P;             // b0 b1 b2  (<= 2^24)
    bm1 = P * q3 + (P - 1u);    // b0 b1 b2 b3 - 1
    uint32_t D = m0 & 0xFFu;
    D = D * q1 + (D + (m1 & 0xFFu));
    D = D * q2 + (D + (m2 & 0xFFu));
    dg = D * q3 + (D + (m3 & 0xFFu));
}

// 32x32 -> 64 multiply-add returning the two halves (forces 32-bit compares
// on the high word instead of a 64-bit compare).
__device__ __forceinline__ void mad_wide(uint32_t a, uint32_t b, uint32_t c_lo, uint32_t c_hi, uint32_t &lo,
                                         uint32_t &hi)
{
    asm("{\n.reg .u64 t, c;\n"
        "mov.b64 c, {%2, %3};\n"
        "mad.wide.u32 t, %4, %5, c;\n"
        "mov.b64 {%0, %1}, t;\n}"
        : "=r"(lo), "=r"(hi)
        : "r"(c_lo), "r"(c_hi), "r"(a), "r"(b));
}

// d*B + D with B-1 = bm1 (< 2^32), d < 2^32, D < 2^32: d*bm1 + (d + D).
__device__ __forceinline__ void fold(uint32_t d, uint32_t bm1, uint32_t D, uint32_t &lo, uint32_t &hi)
{
    uint32_t s_lo, s_hi;
    asm("add.cc.u32 %0, %2, %3;\naddc.u32 %1, 0, 0;" : "=r"(s_lo), "=r"(s_hi) : "r"(d), "r"(D));
    mad_wide(d, bm1, s_lo, s_hi, lo, hi);
}

// One segment that is not the final one of the slice (some lane folds
// digits).  kHot: every lane is active and not in its last segment (all
// 4 pairs valid, all lanes load/extract), so the per-lane predicates vanish.
template <typename V, bool kDecode, bool kHot, class Src>
__device__ __forceinline__ void full_segment(const KernelArgs &a, const Ctx &C, const V *__restrict__ x,
                                             Src &src, const uint32_t j, const uint32_t n,
                                             const uint32_t nseg, uint32_t &w0, uint32_t &w1, uint32_t &w2,
                                             uint32_t &d, uint32_t &r, uint32_t &cur, uint32_t &col, V &acc,
                                             int64_t &out_pos, const int lane)
{
    using T = ValueTraits<V>;
    using Bits = typename T::Bits;
    const uint32_t FULL = 0xFFFFFFFFu;
    const bool act = kHot || j < nseg;
    const bool notlast = kHot || j + 1 < nseg;
    uint32_t so[8], e[8], ds[4];
    Bits vs[4];
    slot_offsets(w0, w1, w2, so);
#pragma unroll
    for (int p = 0; p < 4; p++) lookup_pair<Bits>(C, so[2 * p], so[2 * p + 1], e[2 * p], e[2 * p + 1], ds[p], vs[p]);
    payload_event<T>(C, src, cur, act, e, ds, vs, lane);
    V xv[4];
#pragma unroll
    for (int p = 0; p < 4; p++) {
        const bool valid = kHot || 8u * j + 2u * p < n;
        if (kHot) {
            col += ds[p];
            if (kDecode) {
                a.dec_cols[out_pos] = (int64_t)col;
                reinterpret_cast<Bits *>(a.dec_vals)[out_pos] = vs[p];
                out_pos++;
            } else {
                xv[p] = __ldg(x + min(col, C.cols_m1));
            }
        } else {
            xv[p] = V(0);
            if (valid) {
                col += ds[p];
                if (kDecode) {
                    a.dec_cols[out_pos] = (int64_t)col;
                    reinterpret_cast<Bits *>(a.dec_vals)[out_pos] = vs[p];
                    out_pos++;
                } else {
                    xv[p] = __ldg(x + min(col, C.cols_m1));
                }
            }
        }
    }
    // mixed-radix checks (container.py:478-497): bases decide load vs extract
    uint32_t bm1a, dga, bm1b, dgb;
    group(e[0], e[1], e[2], e[3], bm1a, dga);
    group(e[4], e[5], e[6], e[7], bm1b, dgb);
    uint32_t r1l, r1h, r2l, r2h;
    mad_wide(r, bm1a, r, 0u, r1l, r1h);
    const bool ext0 = r1h != 0u;
    const uint32_t ra = ext0 ? r1h : r1l;
    mad_wide(ra, bm1b, ra, 0u, r2l, r2h);
    const bool ext1 = r2h != 0u;
    const uint32_t m_ld0 = __ballot_sync(FULL, notlast && !ext0);
    const uint32_t m_ld1 = __ballot_sync(FULL, notlast && !ext1);
    const uint32_t m_nl = kHot ? FULL : __ballot_sync(FULL, notlast);
    const uint32_t c1 = cur + __popc(m_ld0);
    const uint32_t c2 = c1 + __popc(m_ld1);
    const uint32_t lw0 = src(cur + __popc(m_ld0 & C.lt));
    const uint32_t lw1 = src(c1 + __popc(m_ld1 & C.lt));
    const uint32_t lw2 = src(c2 + (kHot ? (uint32_t)lane : __popc(m_nl & C.lt)));
    cur = c2 + (kHot ? 32u : __popc(m_nl));
    if (notlast) {
        uint32_t d1l, d1h, d2l, d2h;
        fold(d, bm1a, dga, d1l, d1h);
        const uint32_t da = ext0 ? d1h : d1l;
        w0 = ext0 ? d1l : lw0;
        fold(da, bm1b, dgb, d2l, d2h);
        w1 = ext1 ? d2l : lw1;
        d = ext1 ? d2h : d2l;
        r = ext1 ? r2h : r2l;
        w2 = lw2;
    }
    if (!kDecode) {
#pragma unroll
        for (int p = 0; p < 4; p++) {
            if (kHot) {
                acc = T::add(acc, T::mul(T::from_bits(vs[p]), xv[p]));
            } else if (8u * j + 2u * p < n) {
                acc = T::add(acc, T::mul(T::from_bits(vs[p]), xv[p]));
            }
        }
    }
}

// Per-lane decoder state carried between segments (and restored from a
// long-slice checkpoint).
template <typename V> struct LaneState {
    uint32_t w0, w1, w2, d, r, col, cur;
    V acc;
    int64_t out_pos;
};

// The slice's final segment: every active lane is in its last segment, so
// no digits are folded and no checks/unconditional loads happen.  NP = pairs
// with any valid position in the warp (compile-time, so no per-pair
// branches); slots past them are pads that only matter if they can escape,
// in which case the caller passes NP = 4.
template <typename V, bool kDecode, int NP, class Src>
__device__ __forceinline__ void final_segment(const KernelArgs &a, const Ctx &C, const V *__restrict__ x, Src &src,
                                              const uint32_t jf, const uint32_t n, const uint32_t maxn,
                                              LaneState<V> &st, const int lane)
{
    using T = ValueTraits<V>;
    using Bits = typename T::Bits;
    const bool act = jf < ((n + 7u) >> 3);
    uint32_t so[8], e[8], ds[4];
    Bits vs[4];
    slot_offsets(st.w0, st.w1, st.w2, so);
#pragma unroll
    for (int p = 0; p < 4; p++) {
        if (p < NP) {
            lookup_pair<Bits>(C, so[2 * p], so[2 * p + 1], e[2 * p], e[2 * p + 1], ds[p], vs[p]);
        } else {
            e[2 * p] = e[2 * p + 1] = 0u;
            ds[p] = 0u;
            vs[p] = 0;
        }
    }
    payload_event<T>(C, src, st.cur, act, e, ds, vs, lane);
    const uint32_t base = 8u * jf;
#pragma unroll
    for (int p = 0; p < NP; p++) {
        if (base + 2u * p < n) {
            st.col += ds[p];
            if (kDecode) {
                a.dec_cols[st.out_pos] = (int64_t)st.col;
                reinterpret_cast<Bits *>(a.dec_vals)[st.out_pos] = vs[p];
                st.out_pos++;
            } else {
                const V xv = __ldg(x + min(st.col, C.cols_m1));
                st.acc = T::add(st.acc, T::mul(T::from_bits(vs[p]), xv));
            }
        }
    }
    (void)maxn;
}

// Segments [j0, j1) of a slice (j1 <= max_nseg).  If j1 == max_nseg the
// last one is the final segment: every active lane is in its last segment,
// so no digits are folded and no checks/unconditional loads happen, and
// pairs past the longest row are skipped (pads need lookups only when they
// may escape).  Returns false if the cursor ran past `end` (corrupt slice).
template <typename V, bool kDecode, class Src>
__device__ __forceinline__ bool decode_range(const KernelArgs &a, const Ctx &C, const V *__restrict__ x,
                                             Src &src, const uint32_t end, const uint32_t n,
                                             const uint32_t maxn, const uint32_t j0, const uint32_t j1,
                                             LaneState<V> &st, const int lane)
{
    using T = ValueTraits<V>;
    using Bits = typename T::Bits;
    const uint32_t FULL = 0xFFFFFFFFu;
    const uint32_t nseg = (n + 7u) >> 3;
    const uint32_t max_nseg = (maxn + 7u) >> 3;
    const uint32_t min_nseg = __reduce_min_sync(FULL, nseg);
    const uint32_t jfull = min(j1, max_nseg - 1u);  // segments that fold digits: [j0, jfull)
    // segments where every lane is active and folds digits, then segments
    // where some lane does (per-lane predicates)
    uint32_t j = j0;
    const uint32_t jhot = min(jfull, min_nseg > 0 ? min_nseg - 1u : 0u);
    for (; j < jhot; j++) {
        src.advance(st.cur, lane);
        full_segment<V, kDecode, true>(a, C, x, src, j, n, nseg, st.w0, st.w1, st.w2, st.d, st.r, st.cur, st.col,
                                       st.acc, st.out_pos, lane);
        if (st.cur > end) return false;  // uniform
    }
    for (; j < jfull; j++) {
        src.advance(st.cur, lane);
        full_segment<V, kDecode, false>(a, C, x, src, j, n, nseg, st.w0, st.w1, st.w2, st.d, st.r, st.cur,
                                        st.col, st.acc, st.out_pos, lane);
        if (st.cur > end) return false;
    }
    if (j1 == max_nseg && max_nseg > 0) {
        src.advance(st.cur, lane);
        // pairs the final segment needs: (maxn - 8 jf) / 2 (n is even); all 4
        // lookups are needed only when pads may escape (escape-only table)
        const uint32_t jf = max_nseg - 1;
        const uint32_t np = C.pads_ok ? (maxn - 8u * jf) >> 1 : 4u;
        switch (np) {  // uniform
        case 1: final_segment<V, kDecode, 1>(a, C, x, src, jf, n, maxn, st, lane); break;
        case 2: final_segment<V, kDecode, 2>(a, C, x, src, jf, n, maxn, st, lane); break;
        case 3: final_segment<V, kDecode, 3>(a, C, x, src, jf, n, maxn, st, lane); break;
        default: final_segment<V, kDecode, 4>(a, C, x, src, jf, n, maxn, st, lane); break;
        }
    }
    return true;
}

// init events (container.py:426-429): 3 words per active lane
template <typename V, class Src>
__device__ __forceinline__ void init_state(const Ctx &C, Src &src, const uint32_t n, LaneState<V> &st)
{
    const uint32_t am = __ballot_sync(0xFFFFFFFFu, n > 0);
    const uint32_t cnt = __popc(am), rk = __popc(am & C.lt);
    st.w0 = st.w1 = st.w2 = 0;
    if (n > 0) {
        st.w0 = src(rk);
        st.w1 = src(cnt + rk);
        st.w2 = src(2 * cnt + rk);
    }
    st.cur = 3 * cnt;
    st.d = 0;
    st.r = 1;
    st.col = 0;
    st.acc = V(0);
}

// consumption check (container.py:499-500) and column bound, one vote
__device__ __forceinline__ void report(const KernelArgs &a, const Ctx &C, bool ok, uint32_t cur, uint32_t end,
                                       uint32_t n, uint32_t col, int lane)
{
    const bool col_bad = n > 0 && col > C.cols_m1;
    const bool cur_bad = !ok || cur != end;
    if (__any_sync(0xFFFFFFFFu, col_bad || cur_bad)) {  // rare: report once per slice
        const uint32_t cb = __ballot_sync(0xFFFFFFFFu, col_bad);
        if (lane == 0) atomicOr(a.err, (cur_bad ? 1u : 0u) | (cb ? 2u : 0u));
    }
}

template <typename V, bool kDecode, bool kHasY, class Src>
__device__ __forceinline__ void decode_slice(const KernelArgs &a, const Ctx &C, const V *__restrict__ x,
                                             Src src, const uint32_t end, const uint32_t n,
                                             const uint32_t row, const bool inrow, const int lane)
{
    using T = ValueTraits<V>;
    const uint32_t maxn = __reduce_max_sync(0xFFFFFFFFu, n);
    const uint32_t max_nseg = (maxn + 7u) >> 3;
    if (max_nseg > a.long_seg) return;  // task-decoded slice (uniform)
    const uint32_t orow = (a.row_map != nullptr && inrow) ? __ldg(a.row_map + row) : row;
    V yv = V(0);
    if (kHasY) yv = __ldg(reinterpret_cast<const V *>(a.y) + (inrow ? orow : 0u));
    LaneState<V> st;
    st.out_pos = 0;
    if (kDecode && inrow) st.out_pos = __ldg(a.row_start + row);
    init_state<V>(C, src, n, st);
    const bool ok = decode_range<V, kDecode>(a, C, x, src, end, n, maxn, 0u, max_nseg, st, lane);
    report(a, C, ok, st.cur, end, n, st.col, lane);
    if (!kDecode && inrow) {
        const V res = kHasY ? T::add(st.acc, yv) : st.acc;
        reinterpret_cast<V *>(a.out)[orow] = res;
    }
}

// Long-slice tasks: each warp decodes segments [j0, j1) of one slice from a
// checkpoint (or the init events), reading the stream from global memory,
// and writes its 32 per-lane partial sums (or, when decoding, the columns
// and value bits of those segments directly).
template <typename V, bool kDecode>
__global__ void __launch_bounds__(512, 2) dtans_task_kernel(const KernelArgs a)
{
    using Bits = typename ValueTraits<V>::Bits;
    extern __shared__ __align__(128) unsigned char smem[];
    {
        const int4 *srcv = reinterpret_cast<const int4 *>(a.tables);
        int4 *dst = reinterpret_cast<int4 *>(smem);
        for (int i = threadIdx.x; i < a.table_bytes / 16; i += blockDim.x) dst[i] = __ldg(srcv + i);
    }
    __syncthreads();
    const uint32_t sbase = smem_u32(smem);
    Ctx C;
    C.dtab = sbase;
    C.vtab = sbase + kSlots * 4;
    C.ddict = sbase + (uint32_t)a.off_ddict;
    C.vdict = sbase + (uint32_t)a.off_vdict;
    C.desc_min = a.desc_min;
    C.vesc_min = a.vesc_min;
    C.cols_m1 = (uint32_t)(a.cols - 1);
    C.lt = lanemask_lt();
    C.pads_ok = a.pads_ok != 0;
    const V *__restrict__ x = reinterpret_cast<const V *>(a.x);
    const int lane = threadIdx.x & 31;
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t warps = blockDim.x >> 5;
    for (uint32_t t = blockIdx.x * warps + warp; t < a.ntasks; t += gridDim.x * warps) {
        const LongTask tk = a.tasks[t];
        const uint32_t row = tk.slice * kSliceRows + lane;
        const bool inrow = row < (uint32_t)a.rows;
        const uint32_t n = inrow ? __ldg(a.row_symbols + row) : 0u;
        const uint32_t maxn = __reduce_max_sync(0xFFFFFFFFu, n);
        const uint64_t lo = __ldg(a.directory + tk.slice);
        GmemSrc src{a.stream + lo};
        LaneState<V> st;
        st.out_pos = 0;
        if (tk.ck == 0xFFFFFFFFu) {
            init_state<V>(C, src, n, st);
        } else {
            const uint32_t mask = __ldg(a.ck_pool + tk.ck);
            const bool active = (mask >> lane) & 1u;
            const uint32_t *p = a.ck_pool + tk.ck + 1 + 6 * __popc(mask & C.lt);
            st.w0 = active ? __ldg(p + 0) : 0u;
            st.w1 = active ? __ldg(p + 1) : 0u;
            st.w2 = active ? __ldg(p + 2) : 0u;
            st.d = active ? __ldg(p + 3) : 0u;
            st.r = active ? __ldg(p + 4) : 1u;
            st.col = active ? __ldg(p + 5) : 0u;
            st.cur = tk.cur0;
            st.acc = V(0);
        }
        // decoding: every segment before j0 of an active lane was full (4 pairs)
        if (kDecode && inrow) st.out_pos = __ldg(a.row_start + row) + 4ll * tk.j0;
        const bool ok = decode_range<V, kDecode>(a, C, x, src, tk.cur1, n, maxn, tk.j0, tk.j1, st, lane);
        report(a, C, ok, st.cur, tk.cur1, tk.last ? n : 0u, st.col, lane);
        if (!kDecode) {
            if (tk.last && tk.j0 == 0) {
                // the slice is this single task: y' = acc + y directly
                if (inrow) {
                    const uint32_t orow = a.row_map != nullptr ? __ldg(a.row_map + row) : row;
                    V res = st.acc;
                    if (a.y != nullptr) res = ValueTraits<V>::add(res, reinterpret_cast<const V *>(a.y)[orow]);
                    reinterpret_cast<V *>(a.out)[orow] = res;
                }
            } else {
                reinterpret_cast<V *>(a.partials)[(size_t)tk.part * 32 + lane] = st.acc;
            }
        }
    }
}

// Solo tasks: one THREAD decodes segments [j0, j1) of the only row still
// active in its long slice.  With a single active lane every event of the
// slice belongs to that row (container.py:406-413 with one lane), so its
// words are consecutive from cur0 and the lockstep ballots reduce to a
// running cursor; 32 independent chunks share a warp.
template <typename V, bool kDecode>
__global__ void __launch_bounds__(256) dtans_solo_kernel(const KernelArgs a)
{
    using T = ValueTraits<V>;
    using Bits = typename T::Bits;
    extern __shared__ __align__(128) unsigned char smem[];
    {
        const int4 *srcv = reinterpret_cast<const int4 *>(a.tables);
        int4 *dst = reinterpret_cast<int4 *>(smem);
        for (int i = threadIdx.x; i < a.table_bytes / 16; i += blockDim.x) dst[i] = __ldg(srcv + i);
    }
    __syncthreads();
    const uint32_t sbase = smem_u32(smem);
    const uint32_t dtab = sbase, vtab = sbase + kSlots * 4;
    const uint32_t ddict = sbase + (uint32_t)a.off_ddict, vdict = sbase + (uint32_t)a.off_vdict;
    const uint32_t cols_m1 = (uint32_t)(a.cols - 1);
    const V *__restrict__ x = reinterpret_cast<const V *>(a.x);
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < a.nsolo; t += gridDim.x * blockDim.x) {
        const SoloTask tk = a.solo[t];
        const uint32_t row = tk.slice * kSliceRows + tk.lane;
        const uint32_t n = __ldg(a.row_symbols + row);
        const uint32_t nseg = (n + 7u) >> 3;
        const uint32_t *__restrict__ st = a.stream + __ldg(a.directory + tk.slice);
        const uint32_t *ck = a.ck_pool + tk.ck;
        uint32_t w0 = __ldg(ck), w1 = __ldg(ck + 1), w2 = __ldg(ck + 2), d = __ldg(ck + 3), r = __ldg(ck + 4);
        uint32_t col = __ldg(ck + 5), cur = tk.cur0;
        int64_t out_pos = kDecode ? __ldg(a.row_start + row) + 4ll * tk.j0 : 0;
        V acc = V(0);
        bool ok = true;
        for (uint32_t j = tk.j0; j < tk.j1; j++) {
            uint32_t so[8], e[8], ds[4];
            Bits vs[4];
            slot_offsets(w0, w1, w2, so);
#pragma unroll
            for (int p = 0; p < 4; p++) {
                e[2 * p] = lds32(dtab + so[2 * p]);
                e[2 * p + 1] = lds32(vtab + so[2 * p + 1]);
                ds[p] = lds32(ddict + (e[2 * p] >> 16));
                vs[p] = lds_bits<Bits>(vdict + (e[2 * p + 1] >> 16));
            }
#pragma unroll
            for (int p = 0; p < 4; p++) {  // payloads in slot order, low word first
                if (e[2 * p] >= a.desc_min) ds[p] = __ldg(st + cur++);
                if (e[2 * p + 1] >= a.vesc_min) {
                    if (T::kPayloadWords == 2) {
                        const uint32_t lo = __ldg(st + cur), hi = __ldg(st + cur + 1);
                        vs[p] = (Bits)(((unsigned long long)hi << 32) | lo);
                    } else {
                        vs[p] = (Bits)__ldg(st + cur);
                    }
                    cur += T::kPayloadWords;
                }
            }
#pragma unroll
            for (int p = 0; p < 4; p++) {
                if (8u * j + 2u * p < n) {
                    col += ds[p];
                    if (kDecode) {
                        a.dec_cols[out_pos] = (int64_t)col;
                        reinterpret_cast<Bits *>(a.dec_vals)[out_pos] = vs[p];
                        out_pos++;
                    } else {
                        acc = T::add(acc, T::mul(T::from_bits(vs[p]), __ldg(x + min(col, cols_m1))));
                    }
                }
            }
            if (j + 1 < nseg) {
                uint32_t bm1a, dga, bm1b, dgb, lo, hi;
                group(e[0], e[1], e[2], e[3], bm1a, dga);
                group(e[4], e[5], e[6], e[7], bm1b, dgb);
                mad_wide(r, bm1a, r, 0u, lo, hi);
                uint32_t dl, dh;
                fold(d, bm1a, dga, dl, dh);
                if (hi) {
                    w0 = dl;
                    d = dh;
                    r = hi;
                } else {
                    w0 = __ldg(st + cur++);
                    d = dl;
                    r = lo;
                }
                mad_wide(r, bm1b, r, 0u, lo, hi);
                fold(d, bm1b, dgb, dl, dh);
                if (hi) {
                    w1 = dl;
                    d = dh;
                    r = hi;
                } else {
                    w1 = __ldg(st + cur++);
                    d = dl;
                    r = lo;
                }
                w2 = __ldg(st + cur++);
            }
            if (cur > tk.cur1) {
                ok = false;
                break;
            }
        }
        if (!ok || cur != tk.cur1 || (tk.j1 == nseg && col > cols_m1)) atomicOr(a.err, !ok || cur != tk.cur1 ? 1u : 2u);
        if (!kDecode) reinterpret_cast<V *>(a.partials)[(size_t)tk.part * 32 + tk.lane] = acc;
    }
}

// Long-slice rows: y' = (sum of the row's task partials) + y, in a fixed
// order so the result is deterministic.  Each CTA of 8 warps takes 8 slices
// (warp = slice, lane = row) when the slices have <= 32 partials; a slice
// with more (a long row split into many tasks) gets the whole CTA: warp w
// adds the partials k = w, w+8, ... and the 8 warp sums are added in warp
// order.  Slices made of a single task wrote y' directly (task kernel).
template <typename V, bool kHasY>
__global__ void __launch_bounds__(256) dtans_finalize_kernel(const KernelArgs a)
{
    using T = ValueTraits<V>;
    __shared__ V red[8][32];
    const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
    const V *parts = reinterpret_cast<const V *>(a.partials);
    auto finish = [&](const LongSlice &ls, V s) {
        const uint32_t row = ls.slice * kSliceRows + lane;
        if (row < (uint32_t)a.rows) {
            const uint32_t orow = a.row_map != nullptr ? __ldg(a.row_map + row) : row;
            if (kHasY) s = T::add(s, reinterpret_cast<const V *>(a.y)[orow]);
            reinterpret_cast<V *>(a.out)[orow] = s;
        }
    };
    if (blockIdx.x < a.nlong_small_blocks) {
        const uint32_t i = blockIdx.x * 8u + w;
        if (i >= a.nlong_small) return;
        const LongSlice ls = a.longs[i];
        if (ls.nparts <= 1 && a.single_direct) return;  // written by the task kernel
        const V *part = parts + (size_t)ls.part_base * 32 + lane;
        V acc = part[0];
        for (uint32_t k = 1; k < ls.nparts; k++) acc = T::add(acc, part[(size_t)k * 32]);
        finish(ls, acc);
        return;
    }
    const LongSlice ls = a.longs[a.nlong_small + (blockIdx.x - a.nlong_small_blocks)];
    const V *part = parts + (size_t)ls.part_base * 32 + lane;
    V acc = V(0);
    uint32_t k = w;
    for (; k + 24 < ls.nparts; k += 32) {
        const V p0 = part[(size_t)k * 32], p1 = part[(size_t)(k + 8) * 32];
        const V p2 = part[(size_t)(k + 16) * 32], p3 = part[(size_t)(k + 24) * 32];
        acc = T::add(acc, T::add(T::add(p0, p1), T::add(p2, p3)));
    }
    for (; k < ls.nparts; k += 8) acc = T::add(acc, part[(size_t)k * 32]);
    red[w][lane] = acc;
    __syncthreads();
    if (w == 0) {
        V s = red[0][lane];
#pragma unroll
        for (int q = 1; q < 8; q++) s = T::add(s, red[q][lane]);
        finish(ls, s);
    }
}


// Persistent kernel, one CTA of 32 warps per SM: tables -> shared memory once,
// then every warp walks its slices (grid-wide stride) through its TMA ring.
template <typename V, bool kDecode, bool kHasY, bool kDyn, int kThreads>
__global__ void __launch_bounds__(kThreads, 1) dtans_kernel(const KernelArgs a)
{
    constexpr int kWarps = kThreads / 32;
    extern __shared__ __align__(128) unsigned char smem[];
    {
        const int4 *srcv = reinterpret_cast<const int4 *>(a.tables);
        int4 *dst = reinterpret_cast<int4 *>(smem);
        for (int i = threadIdx.x; i < a.table_bytes / 16; i += blockDim.x) dst[i] = __ldg(srcv + i);
    }
    const uint32_t sbase = smem_u32(smem);
    Ctx C;
    C.dtab = sbase;
    C.vtab = sbase + kSlots * 4;
    C.ddict = sbase + (uint32_t)a.off_ddict;
    C.vdict = sbase + (uint32_t)a.off_vdict;
    C.desc_min = a.desc_min;
    C.vesc_min = a.vesc_min;
    C.cols_m1 = (uint32_t)(a.cols - 1);
    C.lt = lanemask_lt();
    C.pads_ok = a.pads_ok != 0;
    const V *__restrict__ x = reinterpret_cast<const V *>(a.x);
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + a.off_bars) + warp * kRing;
    SliceMeta *meta = reinterpret_cast<SliceMeta *>(smem + a.off_meta) + warp * kRing;
    uint32_t *bufs = reinterpret_cast<uint32_t *>(smem + a.off_bufs) + (size_t)warp * kRing * a.bufw;
    if (lane == 0) {
        for (int b = 0; b < kRing; b++) mbar_init(&bars[b], 1);
        fence_mbar_init();
    }
    __syncthreads();

    const uint32_t rows = (uint32_t)a.rows;  // < 2^32 (checked at upload)
    const uint32_t stride = gridDim.x * kWarps;
    if constexpr (!kDyn) {
        const uint32_t nsl = a.slice_hi;
        const uint32_t first = a.slice_lo + blockIdx.x * kWarps + warp;
        // static order: slices first, first + stride, ...
        if (lane == 0)
            for (int b = 0; b < kRing; b++) {
                const uint32_t s = first + b * stride;
                if (s < nsl)
                    stage_slice(a, s, __ldg(a.directory + s), __ldg(a.directory + s + 1), &bars[b], &meta[b],
                                bufs + b * a.bufw);
            }
        uint32_t n_next = 0;
        if (first < nsl && first * kSliceRows + lane < rows)
            n_next = __ldg(a.row_symbols + first * kSliceRows + lane);
        int b = 0;
        uint32_t parity = 0;
        for (uint32_t s = first; s < nsl; s += stride) {
            const uint32_t n = n_next;
            const uint32_t sn = s + stride;
            n_next = (sn < nsl && sn * kSliceRows + lane < rows) ? __ldg(a.row_symbols + sn * kSliceRows + lane) : 0u;
            // directory entries of the slice this buffer is refilled with
            const uint32_t sr = s + kRing * stride;
            uint64_t rlo = 0, rhi = 0;
            if (lane == 0 && sr < nsl) {
                rlo = __ldg(a.directory + sr);
                rhi = __ldg(a.directory + sr + 1);
            }
            mbar_wait(&bars[b], parity);
            const SliceMeta md = meta[b];
            const uint32_t row = s * kSliceRows + lane;
            const bool inrow = row < rows;
            const uint32_t aw = ((md.off & ~kGlobalSlice) + md.nwords + 3u) & ~3u;  // aligned window
            if (aw > a.long_words) {
                // task-decoded slice (checkpoints.cpp criterion)
            } else if (!(md.off & kGlobalSlice)) {
                const SmemSrc src{smem_u32(bufs + b * a.bufw) + md.off * 4u};
                decode_slice<V, kDecode, kHasY>(a, C, x, src, md.nwords, n, row, inrow, lane);
            } else {
                const GmemSrc src{a.stream + __ldg(a.directory + s)};
                decode_slice<V, kDecode, kHasY>(a, C, x, src, md.nwords, n, row, inrow, lane);
            }
            __syncwarp();
            if (lane == 0 && sr < nsl) stage_slice(a, sr, rlo, rhi, &bars[b], &meta[b], bufs + b * a.bufw);
            if (++b == kRing) {
                b = 0;
                parity ^= 1u;
            }
        }
        return;
    }
    const uint32_t nsl = (uint32_t)a.nslices;
    // Dynamic order (skewed containers): each claim takes the next ticket of
    // a global counter, in the longest-first order of a.slice_order; tickets
    // are claimed kRing slices before they are decoded, so the atomic's
    // latency is hidden.
    auto claim = [&]() -> uint32_t {  // lane 0 only
        const uint32_t p = atomicAdd(a.work_counter, 1u);
        if (p >= nsl) return kNoSlice;
        return a.slice_order != nullptr ? __ldg(a.slice_order + p) : p;
    };
    if (lane == 0) {
        for (int b = 0; b < kRing; b++) {
            const uint32_t s = claim();
            const uint64_t lo = s != kNoSlice ? __ldg(a.directory + s) : 0, hi = s != kNoSlice ? __ldg(a.directory + s + 1) : 0;
            stage_slice(a, s, lo, hi, &bars[b], &meta[b], bufs + b * a.bufw);
        }
    }
    __syncwarp();
    uint32_t s_next = meta[0].slice;
    uint32_t n_next = (s_next != kNoSlice && s_next * kSliceRows + lane < rows)
                          ? __ldg(a.row_symbols + s_next * kSliceRows + lane)
                          : 0u;
    int b = 0;
    uint32_t parity = 0;
    for (;;) {
        // claim the slice this buffer is refilled with, prefetch its directory entries
        uint32_t sr = kNoSlice;
        uint64_t rlo = 0, rhi = 0;
        if (lane == 0) {
            sr = claim();
            if (sr != kNoSlice) {
                rlo = __ldg(a.directory + sr);
                rhi = __ldg(a.directory + sr + 1);
            }
        }
        mbar_wait(&bars[b], parity);
        const SliceMeta md = meta[b];
        const uint32_t s = md.slice;
        if (s == kNoSlice) break;  // uniform
        const uint32_t n = n_next;
        const int bn = b + 1 == kRing ? 0 : b + 1;
        s_next = meta[bn].slice;
        n_next = (s_next != kNoSlice && s_next * kSliceRows + lane < rows)
                     ? __ldg(a.row_symbols + s_next * kSliceRows + lane)
                     : 0u;
        const uint32_t row = s * kSliceRows + lane;
        const bool inrow = row < rows;
        const uint32_t aw = ((md.off & ~kGlobalSlice) + md.nwords + 3u) & ~3u;  // aligned window
        if (aw > a.long_words) {
            // task-decoded slice (checkpoints.cpp criterion)
        } else if (!(md.off & kGlobalSlice)) {
            const SmemSrc src{smem_u32(bufs + b * a.bufw) + md.off * 4u};
            decode_slice<V, kDecode, kHasY>(a, C, x, src, md.nwords, n, row, inrow, lane);
        } else {
            const GmemSrc src{a.stream + __ldg(a.directory + s)};
            decode_slice<V, kDecode, kHasY>(a, C, x, src, md.nwords, n, row, inrow, lane);
        }
        __syncwarp();
        if (lane == 0) stage_slice(a, sr, rlo, rhi, &bars[b], &meta[b], bufs + b * a.bufw);
        __syncwarp();
        b = bn;
        if (b == 0) parity ^= 1u;
    }
}

}  // namespace dev
}  // namespace dtans
