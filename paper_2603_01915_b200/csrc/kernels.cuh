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
// Work unit: a chunk = a run of consecutive slices (host-built list, sized
// to a staging buffer).  Each warp owns a ring of shared-memory buffers;
// lane 0 stages a chunk with three cp.async.bulk copies (TMA bulk engine)
// completing on one mbarrier: the chunk's directory entries, its
// row_symbols, and the 16-byte aligned stream window [dir[s0], dir[s0+k]).
// The decoder then reads everything except x, y and the output from shared
// memory.  Slices that do not fit a buffer (or whose rows are very long) are
// "long" slices, decoded by the checkpointed task kernels instead.
//
// Shared-memory tables.  The two 4096-entry slot tables sit at fixed
// offsets 0 and 16384 (compile-time immediates in LDS), entries
// {digit:8, base-1:8, F:16}.  F is the byte offset of the slot's symbol in
// its dictionary, or, for the delta domain when every retained delta is
// < 0xFFFF, the delta itself ("inline" deltas: no dictionary access).  The
// dictionaries are replicated R times, element e of copy c at (e*R + c)*w
// bytes, and lane i reads copy i % R: with R = 16 (f64) / 32 (f32) a warp's
// 32 random dictionary reads are bank-conflict free.
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
#include <type_traits>

#include "checkpoints.h"

// Build-time switches for A/B experiments (DESIGN 5c); the defaults are the product.
#ifndef DTANS_LATE_VS
#define DTANS_LATE_VS 0  // 1: f64 value-dictionary loads after the escape probe (Laplacian +7%: off)
#endif
#ifndef DTANS_LAG
#define DTANS_LAG 0  // 1: lagged accumulation of hot segments (R-MAT +2.8%, spills: off)
#endif
#ifndef DTANS_MEDIUM
#define DTANS_MEDIUM 1  // the medium payload path (f64: every lane <= two escaped deltas)
#endif
#ifndef DTANS_RORDER
// next-state loads issued before the column prefix and the x gathers:
// 1 in the task kernel (global-memory words) and in pending-products
// segments, 2 everywhere, 0 nowhere (R-MAT sorted -1.1 %, natural -1.0 %,
// Laplacian -0.9 %; banded-27 +0.7 % with 2)
#define DTANS_RORDER 1
#endif
#ifndef DTANS_TICKET_BATCH
#define DTANS_TICKET_BATCH 1  // task kernel: one ticket per pair of tasks (R-MAT sorted -1.3 %, natural +0.4 %)
#endif
#ifndef DTANS_EMPTY_UNROLL
#define DTANS_EMPTY_UNROLL 4  // empty slices in flight per warp (dtans_empty_kernel)
#endif
#ifndef DTANS_PEND2
#define DTANS_PEND2 1  // the pending-products instantiation's direct path for 2-segment uniform slices
#endif
#ifndef DTANS_GMEM_CS
#define DTANS_GMEM_CS 0  // long-slice word loads: 0 L2 evict-first policy, 1 .cs (R-MAT +2.5%), 2 L1::evict_last, 3 __ldg
#endif

namespace dtans {
namespace dev {

constexpr int kSliceRows = 32;
constexpr int kSlots = 4096;
#ifndef DTANS_TASK_WARPS
#define DTANS_TASK_WARPS 32
#endif
constexpr int kMaxWarps = 32;  // warps per CTA of the main kernel
constexpr int kMaxRing = 2;     // staging buffers per warp (a double-buffered ring)
constexpr int kMaxChunk = 16;   // slices per chunk
constexpr uint32_t kTabBytes = 2 * kSlots * 4;
constexpr uint32_t kDeltaInlineEsc = 0xFFFF0000u;  // inline deltas: F = 0xFFFF marks an escape

extern __shared__ __align__(1024) unsigned char dtans_smem[];

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

// A chunk: slices [s0, s0 + k) (k = kw & 0xFF) stored as one contiguous
// blob of kw >> 8 words at word offset `off` of the chunk-blob array:
//   [next: the ChunkRec this warp stages into the same buffer after this
//    chunk (chunk index + 2 x the static stride), zero when none or when the
//    plan is dynamic][hdr: k u32 slice words, padded to 4]
//   [row_symbols: k*32 u32][stream words, padded to 4]
// hdr[i] describes slice s0+i (host-computed once at upload, slice_meta()):
//   bits  0-15  directory[s0+i+1] - directory[s0]: the end of the slice's
//               words relative to the chunk (container.py:296-317); the
//               start is the previous slice's end (0 for i = 0)
//   bits 16-22  max_nseg  = ceil(max row_symbols / 8) over the slice's 32 rows
//   bits 23-29  min_nseg  (rows past the matrix count as 0)
//   bits 30-31  np - 1: pairs the final segment decodes (4 if pads may escape)
// so the per-slice warp reductions and final-segment arithmetic are paid once
// on the host instead of once per slice per SpMV.
struct __align__(16) ChunkRec {
    unsigned long long off;
    uint32_t s0;
    uint32_t kw;
};
// words before a chunk's row_symbols: the embedded next record (4 words),
// then the k slice words padded to 4
__host__ __device__ constexpr uint32_t chunk_hdr_words(uint32_t k) { return 4u + ((k + 3u) & ~3u); }
constexpr uint32_t kMetaMaxNseg = 127u;  // max_nseg field width (7 bits)
__host__ __device__ constexpr uint32_t slice_meta(uint32_t end_rel, uint32_t max_nseg, uint32_t min_nseg,
                                                  uint32_t np)
{
    return end_rel | (max_nseg << 16) | (min_nseg << 23) | ((np - 1u) & 3u) << 30;
}

struct KernelArgs {
    const uint32_t *tables;       // shared-memory image [off_img, off_img + table_bytes) (global copy)
    int32_t table_bytes;          // bytes to copy into shared memory (multiple of 16)
    int32_t off_img, off_tab;     // image start; delta slot table (16 KB aligned address), value table +16 KB
    int32_t off_ddict, off_vdict; // byte offsets in shared memory (replicated dictionaries)
    int32_t rep_d, rep_v;         // replication factors (powers of two)
    uint32_t desc_min, vesc_min;  // entry >= this  <=>  escape
    int32_t pads_ok;              // both domains retain a pad symbol
    int32_t off_bars, off_meta, off_ctl, off_bufs;  // shared-memory layout
    int32_t bufb;                 // bytes per staging buffer (multiple of 16)
    int32_t nring;                // staging buffers per warp (kMaxRing)
    const uint32_t *blob;         // chunk blobs (main kernel)
    const uint32_t *row_symbols;  // rows (long-slice kernels only)
    const uint64_t *directory;    // nslices + 1 (long-slice kernels only)
    const uint32_t *stream;       // nwords + kStreamPadWords (long-slice kernels only)
    int64_t rows, cols, nslices, nwords;
    const void *x;
    const void *y;                // may be null (y' = A x)
    void *out;
    const int64_t *row_start;     // decode kernel only
    int64_t *dec_cols;            // decode kernel only
    void *dec_vals;               // decode kernel only
    unsigned int *err;            // bit 0: consumption mismatch, bit 1: column OOB
    // long slices (checkpoint index, checkpoints.cpp)
    uint32_t ntasks, nlong, nsolo;
    uint32_t nlong_small, nlong_small_blocks;  // finalize: slices with <= 32 partials come first
    int32_t single_direct;                      // single-task slices write y' in the task kernel
    int32_t task_dyn;                           // task kernel: atomic tickets after the first round
    const LongTask *tasks;
    const SoloTask *solo;
    const uint32_t *ck_pool;
    const LongSlice *longs;
    void *partials;               // V[nparts][32]
    const uint32_t *row_map;      // optional: y/out index of encoded row i (row-reordered P*A)
    // power iteration (scaled kernel): out = (A x) / sqrt(*sumsq_in), *sumsq_out += sum(out^2)
    const double *sumsq_in;       // null: no scaling
    double *sumsq_out;
    double *sumsq_zero;           // zeroed by the kernel (the accumulator of the next iteration)
    // work distribution over the chunk list
    const ChunkRec *chunks;
    uint32_t chunk_lo, chunk_hi;  // chunks of this launch
    int32_t dynamic;              // 1: atomic ticket counter instead of a static stride
    uint32_t embed_stride;        // static stride (CTAs x warps) the blobs' next records were built for; 0: none
    int32_t work_warps;           // main kernel: warps per CTA that decode (the CTA always has kMaxWarps)
    uint32_t *work_counter;       // zeroed before every dynamic launch
    // all-empty slices of a long-slice plan (y' = +0.0 + y), outside the chunk list
    const uint32_t *empty_slices;
    uint32_t nempty;
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

// Shared-memory loads at absolute 32-bit shared addresses (ld.shared with
// a register + immediate address).
__device__ __forceinline__ uint32_t sh32(uint32_t addr)
{
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long sh64(uint32_t addr)
{
    unsigned long long v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(addr) : "memory");
    return v;
}
// Tables and dictionaries never change after the CTA prologue: plain
// (non-volatile) loads the compiler may schedule freely.
__device__ __forceinline__ uint32_t tab32(uint32_t addr)
{
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t vtab32(uint32_t addr)
{
    uint32_t v;
    asm("ld.shared.u32 %0, [%1+16384];" : "=r"(v) : "r"(addr));
    return v;
}
template <typename Bits> __device__ __forceinline__ Bits dict_bits(uint32_t addr);
template <> __device__ __forceinline__ unsigned long long dict_bits<unsigned long long>(uint32_t addr)
{
    unsigned long long v;
    asm("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(addr));
    return v;
}
template <> __device__ __forceinline__ uint32_t dict_bits<uint32_t>(uint32_t addr) { return tab32(addr); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar)
{
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

// Streamed container bytes are read exactly once per SpMV: mark them
// evict-first in L2 so they do not push out x, which is gathered repeatedly.
__device__ __forceinline__ unsigned long long policy_evict_first()
{
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void bulk_g2s_stream(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar)
{
    asm volatile(
        "{\n.reg .b64 pol;\n"
        "createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], pol;\n}"
        ::"r"(dst), "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

// Programmatic dependent launch (api.cu launch_pdl): the main, task and
// solo kernels let the next kernel of the chain start on the SMs they free
// (their tails overlap); the task and solo kernels do not read the main
// kernel's output, so they only wait for their predecessor at the very end
// (their completion then implies its completion, which keeps the stream
// order for everything after the chain); finalize waits up front (it reads
// the partials).  Both are no-ops in a kernel launched without PDL.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void fence_mbar_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Word sources for one slice, addressed by the position relative to
// directory[s] (32-bit): the staged shared-memory window or global memory.
// Reads are not clamped: a segment consumes at most kSegMaxWords words, the
// decoder stops as soon as its cursor passes the slice end (then reports
// CorruptStream), and both the staging buffers and the device stream carry
// at least kOverrunWords of slack, so a corrupt container can never read
// outside the allocations.
constexpr uint32_t kSegMaxWords = 32u * 15u;  // payload 12 + 2 checks + 1 uncond per lane
constexpr uint32_t kOverrunWords = 3u * 32u + kSegMaxWords + 64u;
constexpr uint32_t kStreamPadWords = kOverrunWords;  // device stream padding
struct SmemSrc {
    uint32_t addr;  // shared address of word directory[s]
    __device__ __forceinline__ uint32_t operator()(uint32_t rel) const { return sh32(addr + rel * 4u); }
    __device__ __forceinline__ void prepare(uint32_t) {}
};
struct GmemSrc {
    const uint32_t *p;  // the task's first word
#if DTANS_GMEM_CS == 1
    // ld.global.cs.nc: evict-first in L1 and L2, no cache-policy register
    __device__ __forceinline__ uint32_t at(const uint32_t *q) const
    {
        uint32_t v;
        asm("ld.global.cs.nc.u32 %0, [%1];" : "=r"(v) : "l"(q));
        return v;
    }
#elif DTANS_GMEM_CS == 2
    // ld.global.nc.L1::evict_last: the prefetched words stay in L1
    __device__ __forceinline__ uint32_t at(const uint32_t *q) const
    {
        uint32_t v;
        asm("ld.global.nc.L1::evict_last.u32 %0, [%1];" : "=r"(v) : "l"(q));
        return v;
    }
#elif DTANS_GMEM_CS == 3
    __device__ __forceinline__ uint32_t at(const uint32_t *q) const { return __ldg(q); }
#else
    unsigned long long pol;  // L2 evict-first policy (streamed words)
    __device__ __forceinline__ uint32_t at(const uint32_t *q) const
    {
        uint32_t v;
        asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(q), "l"(pol));
        return v;
    }
#endif
    __device__ __forceinline__ uint32_t operator()(uint32_t rel) const { return at(p + rel); }
    __device__ __forceinline__ void prepare(uint32_t) {}
};

// Per-lane shared-memory context (absolute shared addresses).  The delta
// slot table starts on a 16 KB boundary, so a slot's address is one LOP3:
// (bits & 0x3FFC) | tab; the value table follows at +16384.
struct Ctx {
    uint32_t tab;                       // shared address of the delta slot table
    uint32_t dbase, vbase;              // dictionary + this lane's copy
    uint32_t desc_min, vesc_min;        // entry >= this <=> escape
    uint32_t cols_m1;
    uint32_t lt;                        // lanemask_lt
    bool pads_ok;
};

template <typename V>
__device__ __forceinline__ Ctx make_ctx(const KernelArgs &a, int lane)
{
    const uint32_t sb = smem_u32(dtans_smem);
    Ctx C;
    C.tab = sb + (uint32_t)a.off_tab;
    C.dbase = sb + (uint32_t)a.off_ddict + (uint32_t)(lane & (a.rep_d - 1)) * 4u;
    C.vbase = sb + (uint32_t)a.off_vdict + (uint32_t)(lane & (a.rep_v - 1)) * (uint32_t)sizeof(V);
    C.desc_min = a.desc_min;
    C.vesc_min = a.vesc_min;
    C.cols_m1 = (uint32_t)(a.cols - 1);
    C.lt = lanemask_lt();
    C.pads_ok = a.pads_ok != 0;
    return C;
}

// Copy the table image into shared memory (all threads; caller syncs).
// Returns false if the tables are not 16 KB aligned in the shared window
// (the kernel then reports an error instead of decoding).
__device__ __forceinline__ bool load_tables(const KernelArgs &a)
{
    const int4 *src = reinterpret_cast<const int4 *>(a.tables);
    int4 *dst = reinterpret_cast<int4 *>(dtans_smem + a.off_img);
    for (int i = threadIdx.x; i < a.table_bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
    return ((smem_u32(dtans_smem) + (uint32_t)a.off_tab) & 0x3FFFu) == 0u;
}

__device__ __forceinline__ void slot_offsets(const uint32_t tab, uint32_t w0, uint32_t w1, uint32_t w2,
                                             uint32_t so[8])
{
    // unpack (codec.py:148-162): slot k = bits [12k, 12k+12) of w0:w1:w2, as
    // shared addresses tab + slot * 4 (tab is 16 KB aligned: OR == ADD)
    so[0] = ((w2 << 2) & 0x3FFCu) | tab;
    so[1] = ((w2 >> 10) & 0x3FFCu) | tab;
    so[2] = (__funnelshift_r(w2, w1, 22) & 0x3FFCu) | tab;
    so[3] = ((w1 >> 2) & 0x3FFCu) | tab;
    so[4] = ((w1 >> 14) & 0x3FFCu) | tab;
    so[5] = (__funnelshift_r(w1, w0, 26) & 0x3FFCu) | tab;
    so[6] = ((w0 >> 6) & 0x3FFCu) | tab;
    so[7] = ((w0 >> 18) & 0x3FFCu) | tab;
}

// Table entries of pair p and the symbols they decode to (escape entries
// point at a dummy dictionary slot / carry 0xFFFF; the payload overwrites
// them).
template <typename Bits, bool kDIn>
__device__ __forceinline__ void lookup_pair(const Ctx &C, uint32_t sod, uint32_t sov, uint32_t &ed, uint32_t &ev,
                                            uint32_t &ds, Bits &vs)
{
    ed = tab32(sod);
    ev = vtab32(sov);
    ds = kDIn ? (ed >> 16) : tab32(C.dbase + (ed >> 16));
    vs = dict_bits<Bits>(C.vbase + (ev >> 16));
}

// Payload event (container.py:459-470): per-lane word counts, exclusive warp
// scan, words read in slot order, low word first, overwriting the symbols.
// Split in three so callers can give the general (slow) case its own copy
// of the rest of the segment: the common paths then never merge 64-bit value
// registers (no register shuffling on the hot path).
//   payload_probe: 0 = no escape in the warp, 1 = fast case (every lane needs
//   at most one payload word: its rank among the escaping lanes; f64 value
//   escapes never qualify), 2 = general case.
template <typename T, int NP = 4, bool kMedium = false>
__device__ __forceinline__ int payload_probe(const Ctx &C, const bool act, const uint32_t e[8], bool &dany)
{
    const uint32_t FULL = 0xFFFFFFFFu;
    // cheap test first: escape entries are the largest entries of a table.
    // NP < 4 (final segments): pairs past NP are pads of a table with a pad
    // symbol, never escapes, and are not looked at.
    uint32_t dmax, vmax;
    if (NP == 4) {
        dmax = max(max(e[0], e[2]), max(e[4], e[6]));
        vmax = max(max(e[1], e[3]), max(e[5], e[7]));
    } else if (NP == 3) {
        dmax = max(max(e[0], e[2]), e[4]);
        vmax = max(max(e[1], e[3]), e[5]);
    } else if (NP == 2) {
        dmax = max(e[0], e[2]);
        vmax = max(e[1], e[3]);
    } else {
        dmax = e[0];
        vmax = e[1];
    }
    dany = act && dmax >= C.desc_min;
    const bool vany = act && vmax >= C.vesc_min;
    if (!__any_sync(FULL, dany || vany)) return 0;
    bool fast;
    if (T::kPayloadWords == 2) {
        // f64: no value escape, and at most one delta escape per lane, i.e.
        // the second-largest delta entry does not escape
        uint32_t d2 = 0u;
        if (NP == 4) {
            const uint32_t m02 = max(e[0], e[2]), m46 = max(e[4], e[6]);
            d2 = max(max(min(e[0], e[2]), min(e[4], e[6])), min(m02, m46));
        } else if (NP == 3) {
            d2 = max(min(e[0], e[2]), min(max(e[0], e[2]), e[4]));
        } else if (NP == 2) {
            d2 = min(e[0], e[2]);
        }
        fast = !vany && !(act && d2 >= C.desc_min);
    } else {
        int nd = 0, nv = 0;
#pragma unroll
        for (int p = 0; p < NP; p++) {
            nd += e[2 * p] >= C.desc_min ? 1 : 0;
            nv += e[2 * p + 1] >= C.vesc_min ? 1 : 0;
        }
        fast = !act || nd + nv <= 1;
    }
    if (__all_sync(FULL, fast)) return 1;
    if (kMedium && DTANS_MEDIUM && T::kPayloadWords == 2) {
        // 3 = medium case (f64): every lane needs at most two one-word
        // payloads (two escaped deltas); banded-27 -0.8 %, while for f32
        // (R-MAT: many lanes with more escapes) the extra probe cost +1-5 %
        int nd = 0, nv = 0;
#pragma unroll
        for (int p = 0; p < NP; p++) {
            nd += e[2 * p] >= C.desc_min ? 1 : 0;
            nv += e[2 * p + 1] >= C.vesc_min ? 1 : 0;
        }
        const bool med = !act || (T::kPayloadWords == 2 ? (nv == 0 && nd <= 2) : nd + nv <= 2);
        if (__all_sync(FULL, med)) return 3;
    }
    return 2;
}

// Medium payload event: every lane reads at most two words (one-word
// payloads), at its offset from a two-plane ballot scan; the escaped slots
// take them in slot order.  Two loads instead of one per escaped slot.
template <typename T, class Src>
__device__ __forceinline__ void payload_medium(const Ctx &C, const Src &src, uint32_t &cur, const bool act,
                                               const uint32_t e[8], uint32_t ds[4], typename T::Bits vs[4])
{
    using Bits = typename T::Bits;
    const uint32_t FULL = 0xFFFFFFFFu;
    uint32_t pc = 0;
#pragma unroll
    for (int p = 0; p < 4; p++)
        pc += (e[2 * p] >= C.desc_min ? 1u : 0u) + (T::kPayloadWords == 1 && e[2 * p + 1] >= C.vesc_min ? 1u : 0u);
    if (!act) pc = 0;
    const uint32_t b0 = __ballot_sync(FULL, pc & 1u);
    const uint32_t b1 = __ballot_sync(FULL, pc & 2u);
    const uint32_t off = cur + __popc(b0 & C.lt) + (__popc(b1 & C.lt) << 1);
    cur += __popc(b0) + (__popc(b1) << 1);
    const uint32_t w0 = pc >= 1u ? src(off) : 0u;
    const uint32_t w1 = pc >= 2u ? src(off + 1u) : 0u;
    bool second = false;
#pragma unroll
    for (int p = 0; p < 4; p++) {
        if (e[2 * p] >= C.desc_min) {
            ds[p] = second ? w1 : w0;
            second = true;
        }
        if (T::kPayloadWords == 1 && e[2 * p + 1] >= C.vesc_min) {
            vs[p] = (Bits)(second ? w1 : w0);
            second = true;
        }
    }
}

// Fast payload event: every lane reads at most one word, at its rank among
// the escaping lanes.  f64 (kPayloadWords == 2): only a delta can escape
// here, so `dany` (from the probe) is the lane's escape flag.
template <typename T, class Src, int NP = 4>
__device__ __forceinline__ void payload_fast(const Ctx &C, const Src &src, uint32_t &cur, const bool act,
                                             const bool dany, const uint32_t e[8], uint32_t ds[4],
                                             typename T::Bits vs[4])
{
    using Bits = typename T::Bits;
    bool esc = dany;
    if (T::kPayloadWords == 1) {
#pragma unroll
        for (int p = 0; p < NP; p++) esc = esc || (act && e[2 * p + 1] >= C.vesc_min);
    }
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, esc);
    const uint32_t w = src(cur + __popc(m & C.lt));
    cur += __popc(m);
#pragma unroll
    for (int p = 0; p < NP; p++) {
        if (e[2 * p] >= C.desc_min) ds[p] = w;
        if (T::kPayloadWords == 1 && e[2 * p + 1] >= C.vesc_min) vs[p] = (Bits)w;
    }
}

template <typename T, class Src, int NP = 4>
__device__ __forceinline__ void payload_slow(const Ctx &C, const Src &src, uint32_t &cur, const bool act,
                                             const uint32_t e[8], uint32_t ds[4], typename T::Bits vs[4])
{
    using Bits = typename T::Bits;
    const uint32_t FULL = 0xFFFFFFFFu;
    uint32_t pc = 0;
#pragma unroll
    for (int p = 0; p < NP; p++)
        pc += (e[2 * p] >= C.desc_min ? 1u : 0u) + (e[2 * p + 1] >= C.vesc_min ? (uint32_t)T::kPayloadWords : 0u);
    if (!act) pc = 0;
    // exclusive warp scan of pc (<= 12 words: 4 bit planes), one ballot per
    // plane: independent ballots instead of a dependent 5-step shuffle chain
    const uint32_t b1 = __ballot_sync(FULL, pc & 2u);
    const uint32_t b2 = __ballot_sync(FULL, pc & 4u);
    const uint32_t b3 = __ballot_sync(FULL, pc & 8u);
    const uint32_t b0 = __ballot_sync(FULL, pc & 1u);
    const uint32_t excl = __popc(b0 & C.lt) + (__popc(b1 & C.lt) << 1) + (__popc(b2 & C.lt) << 2) +
                          (__popc(b3 & C.lt) << 3);
    const uint32_t total = __popc(b0) + (__popc(b1) << 1) + (__popc(b2) << 2) + (__popc(b3) << 3);
    if (pc) {
        {
            uint32_t off = cur + excl;
#pragma unroll
            for (int p = 0; p < NP; p++) {
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
    }
    cur += total;
}

// All three in one (final segments and the solo path, where the extra
// copy is not worth it).
template <typename T, class Src, int NP = 4>
__device__ __forceinline__ void payload_event(const Ctx &C, const Src &src, uint32_t &cur, const bool act,
                                              const uint32_t e[8], uint32_t ds[4], typename T::Bits vs[4])
{
    bool dany;
    const int pk = payload_probe<T, NP>(C, act, e, dany);
    if (pk == 1) payload_fast<T, Src, NP>(C, src, cur, act, dany, e, ds, vs);
    else if (pk == 2) payload_slow<T, Src, NP>(C, src, cur, act, e, ds, vs);
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

// d*B + D with B-1 = bm1 (< 2^32), d < 2^32, D < 2^32: (d*bm1 + D) + d.
__device__ __forceinline__ void fold(uint32_t d, uint32_t bm1, uint32_t D, uint32_t &lo, uint32_t &hi)
{
    uint32_t t_lo, t_hi;
    mad_wide(d, bm1, D, 0u, t_lo, t_hi);
    asm("add.cc.u32 %0, %2, %3;\naddc.u32 %1, %4, 0;" : "=r"(lo), "=r"(hi) : "r"(t_lo), "r"(d), "r"(t_hi));
}

// One segment that is not the final one of the slice (some lane folds
// digits).  kHot: every lane is active and not in its last segment (all
// 4 pairs valid, all lanes load/extract), so the per-lane predicates vanish.
// Products of a hot segment whose accumulation is deferred: its four
// value symbols and gathered x, accumulated (in order) by the final segment
// after that segment has issued its own gathers, so the last full segment's
// x latency overlaps the final segment's decode.
template <typename V> struct Pend4 {
    typename ValueTraits<V>::Bits vs[4];
    V xv[4];
};

template <typename V, bool kDecode, bool kHot, bool kDIn, class Src, bool kDefer = false>
__device__ __forceinline__ void full_segment(const KernelArgs &a, const Ctx &C, const V *__restrict__ x,
                                             const Src &src, const uint32_t j, const uint32_t n,
                                             const uint32_t nseg, uint32_t &w0, uint32_t &w1, uint32_t &w2,
                                             uint32_t &d, uint32_t &r, uint32_t &cur, uint32_t &col, V &acc,
                                             int64_t &out_pos, const int lane, Pend4<V> *pd = nullptr)
{
    using T = ValueTraits<V>;
    using Bits = typename T::Bits;
    const uint32_t FULL = 0xFFFFFFFFu;
    const bool act = kHot || j < nseg;
    const bool notlast = kHot || j + 1 < nseg;
    uint32_t so[8], e[8], ds[4];
    Bits vs[4];
    slot_offsets(C.tab, w0, w1, w2, so);
    // f64 (DTANS_LATE_VS): the value symbols are read from the dictionary
    // after the escape probe on the paths where no value escapes (the fast
    // path carries only deltas), so the probe's two paths do not have to
    // keep four 64-bit values in matching registers
    constexpr bool kLate = DTANS_LATE_VS && T::kPayloadWords == 2;
#pragma unroll
    for (int p = 0; p < 4; p++) {
        e[2 * p] = tab32(so[2 * p]);
        e[2 * p + 1] = vtab32(so[2 * p + 1]);
        ds[p] = kDIn ? (e[2 * p] >> 16) : tab32(C.dbase + (e[2 * p] >> 16));
        if (!kLate) vs[p] = dict_bits<Bits>(C.vbase + (e[2 * p + 1] >> 16));
    }
    auto load_vs = [&]() __attribute__((always_inline)) {
#pragma unroll
        for (int p = 0; p < 4; p++) vs[p] = dict_bits<Bits>(C.vbase + (e[2 * p + 1] >> 16));
    };
    // the rest of the segment once the symbols are final
    auto rest = [&](const uint32_t (&ds)[4], const Bits (&vs)[4]) __attribute__((always_inline)) {
        V xv[4];
        auto gathers = [&]() __attribute__((always_inline)) {
#pragma unroll
            for (int p = 0; p < 4; p++) {
                const bool valid = kHot || 8u * j + 2u * p < n;
                xv[p] = V(0);
                if (valid) {
                    col += ds[p];
                    if (kDecode) {
                        if (a.dec_cols != nullptr) {  // null: the checkpoint walk only needs the state
                            a.dec_cols[out_pos] = (int64_t)col;
                            reinterpret_cast<Bits *>(a.dec_vals)[out_pos] = vs[p];
                        }
                        out_pos++;
                    } else {
                        xv[p] = __ldg(x + min(col, C.cols_m1));
                    }
                }
            }
        };
        constexpr bool kRO = DTANS_RORDER == 2 || (DTANS_RORDER == 1 && (kDefer || std::is_same<Src, GmemSrc>::value));
        if (!kRO) gathers();
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
        if (kRO) gathers();
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
        if (kDefer) {
#pragma unroll
            for (int p = 0; p < 4; p++) {
                pd->vs[p] = vs[p];
                pd->xv[p] = xv[p];
            }
        } else if (!kDecode) {
#pragma unroll
            for (int p = 0; p < 4; p++) {
                if (kHot || 8u * j + 2u * p < n) acc = T::add(acc, T::mul(T::from_bits(vs[p]), xv[p]));
            }
        }
    };
    bool dany;
    const int pk = payload_probe<T, 4, true>(C, act, e, dany);
    if (pk == 2) {
        if (kLate) load_vs();
        payload_slow<T>(C, src, cur, act, e, ds, vs);
        rest(ds, vs);
        return;
    }
    if (pk == 1) payload_fast<T>(C, src, cur, act, dany, e, ds, vs);
    else if (pk == 3) payload_medium<T>(C, src, cur, act, e, ds, vs);
    if (kLate) load_vs();
    rest(ds, vs);
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
template <typename V, bool kDecode, bool kDIn, int NP, class Src, bool kPend = false>
__device__ __forceinline__ void final_segment(const KernelArgs &a, const Ctx &C, const V *__restrict__ x,
                                              const Src &src, const uint32_t jf, const uint32_t n,
                                              LaneState<V> &st, const Pend4<V> *pd = nullptr)
{
    using T = ValueTraits<V>;
    using Bits = typename T::Bits;
    const bool act = jf < ((n + 7u) >> 3);
    uint32_t so[8], e[8], ds[4];
    Bits vs[4];
    slot_offsets(C.tab, st.w0, st.w1, st.w2, so);
#pragma unroll
    for (int p = 0; p < 4; p++) {
        if (p < NP) {
            lookup_pair<Bits, kDIn>(C, so[2 * p], so[2 * p + 1], e[2 * p], e[2 * p + 1], ds[p], vs[p]);
        } else {
            e[2 * p] = e[2 * p + 1] = 0u;
            ds[p] = 0u;
            vs[p] = 0;
        }
    }
    // the event over the NP pairs only (pads past them never escape)
    payload_event<T, Src, NP>(C, src, st.cur, act, e, ds, vs);
    const uint32_t base = 8u * jf;
    if (kPend) {
        // gathers first, then the previous segment's products, then ours
        V xv[NP];
#pragma unroll
        for (int p = 0; p < NP; p++) {
            xv[p] = V(0);
            if (base + 2u * p < n) {
                st.col += ds[p];
                xv[p] = __ldg(x + min(st.col, C.cols_m1));
            }
        }
#pragma unroll
        for (int p = 0; p < 4; p++) st.acc = T::add(st.acc, T::mul(T::from_bits(pd->vs[p]), pd->xv[p]));
#pragma unroll
        for (int p = 0; p < NP; p++)
            if (base + 2u * p < n) st.acc = T::add(st.acc, T::mul(T::from_bits(vs[p]), xv[p]));
        return;
    }
#pragma unroll
    for (int p = 0; p < NP; p++) {
        if (base + 2u * p < n) {
            st.col += ds[p];
            if (kDecode) {
                if (a.dec_cols != nullptr) {
                    a.dec_cols[st.out_pos] = (int64_t)st.col;
                    reinterpret_cast<Bits *>(a.dec_vals)[st.out_pos] = vs[p];
                }
                st.out_pos++;
            } else {
                const V xv = __ldg(x + min(st.col, C.cols_m1));
                st.acc = T::add(st.acc, T::mul(T::from_bits(vs[p]), xv));
            }
        }
    }
}

// Segments [j0, j1) of a slice (j1 <= max_nseg).  If j1 == max_nseg the
// last one is the final segment: every active lane is in its last segment,
// so no digits are folded and no checks/unconditional loads happen, and
// pairs past the longest row are skipped (pads need lookups only when they
// may escape).  Returns false if the cursor ran past `end` (corrupt slice).
// kPend (SpMV): when every lane is hot up to a one-pair final segment,
// that segment's gather goes out before the last full segment's products are
// accumulated (Pend4), so the two x latencies overlap.
template <typename V, bool kDecode, bool kDIn, class Src, bool kPend = false>
__device__ __forceinline__ bool decode_range(const KernelArgs &a, const Ctx &C, const V *__restrict__ x,
                                             Src &src, const uint32_t end, const uint32_t n,
                                             const uint32_t max_nseg, const uint32_t min_nseg, const uint32_t np,
                                             const uint32_t j0, const uint32_t j1, LaneState<V> &st, const int lane)
{
    const uint32_t nseg = (n + 7u) >> 3;
    const uint32_t jfull = min(j1, max_nseg - 1u);  // segments that fold digits: [j0, jfull)
    // segments where every lane is active and folds digits, then segments
    // where some lane does (per-lane predicates)
    uint32_t j = j0;
    const uint32_t jhot = min(jfull, min_nseg > 0 ? min_nseg - 1u : 0u);
    if (kPend && !kDecode && j1 == max_nseg && jhot == jfull && jfull > j0 && np == 1u) {
        // hot up to a short final segment: its gathers go out before the
        // last full segment's products are accumulated
        for (; j + 1 < jfull; j++) {
            src.prepare(st.cur);
            full_segment<V, kDecode, true, kDIn>(a, C, x, src, j, n, nseg, st.w0, st.w1, st.w2, st.d, st.r, st.cur,
                                                 st.col, st.acc, st.out_pos, lane);
            if (st.cur > end) return false;  // uniform
        }
        Pend4<V> pd;
        src.prepare(st.cur);
        full_segment<V, kDecode, true, kDIn, Src, !kDecode>(a, C, x, src, j, n, nseg, st.w0, st.w1, st.w2, st.d,
                                                             st.r, st.cur, st.col, st.acc, st.out_pos, lane, &pd);
        if (st.cur > end) return false;
        src.prepare(st.cur);
        final_segment<V, kDecode, kDIn, 1, Src, !kDecode>(a, C, x, src, max_nseg - 1, n, st, &pd);
        return true;
    }
#if DTANS_LAG
    if (!kDecode && !kPend) {
        // lagged accumulation (experiment): each hot segment's products are
        // accumulated after the next segment's gathers are issued
        Pend4<V> pd;
        bool have = false;
        for (; j < jhot; j++) {
            src.prepare(st.cur);
            Pend4<V> cur;
            full_segment<V, kDecode, true, kDIn, Src, true>(a, C, x, src, j, n, nseg, st.w0, st.w1, st.w2, st.d, st.r,
                                                            st.cur, st.col, st.acc, st.out_pos, lane, &cur);
            if (have) {
#pragma unroll
                for (int p = 0; p < 4; p++)
                    st.acc = ValueTraits<V>::add(st.acc, ValueTraits<V>::mul(ValueTraits<V>::from_bits(pd.vs[p]), pd.xv[p]));
            }
            pd = cur;
            have = true;
            if (st.cur > end) return false;  // uniform
        }
        if (have) {
#pragma unroll
            for (int p = 0; p < 4; p++)
                st.acc = ValueTraits<V>::add(st.acc, ValueTraits<V>::mul(ValueTraits<V>::from_bits(pd.vs[p]), pd.xv[p]));
        }
    }
#endif
    for (; j < jhot; j++) {
        src.prepare(st.cur);
        full_segment<V, kDecode, true, kDIn>(a, C, x, src, j, n, nseg, st.w0, st.w1, st.w2, st.d, st.r, st.cur,
                                             st.col, st.acc, st.out_pos, lane);
        if (st.cur > end) return false;  // uniform
    }
    for (; j < jfull; j++) {
        src.prepare(st.cur);
        full_segment<V, kDecode, false, kDIn>(a, C, x, src, j, n, nseg, st.w0, st.w1, st.w2, st.d, st.r,
                                              st.cur, st.col, st.acc, st.out_pos, lane);
        if (st.cur > end) return false;
    }
    if (j1 == max_nseg && max_nseg > 0) {
        // np = pairs the final segment needs (all 4 lookups only when pads
        // may escape: escape-only table)
        const uint32_t jf = max_nseg - 1;
        src.prepare(st.cur);
        switch (np) {  // uniform
        case 1: final_segment<V, kDecode, kDIn, 1>(a, C, x, src, jf, n, st); break;
        case 2: final_segment<V, kDecode, kDIn, 2>(a, C, x, src, jf, n, st); break;
        case 3: final_segment<V, kDecode, kDIn, 3>(a, C, x, src, jf, n, st); break;
        default: final_segment<V, kDecode, kDIn, 4>(a, C, x, src, jf, n, st); break;
        }
    }
    return true;
}

// The slice shape from the lanes' row lengths (long-slice tasks, which have
// no host-built slice metadata): max_nseg, min_nseg and the final segment's
// pair count, as slice_meta() records them for chunked slices.
__device__ __forceinline__ void slice_shape(const Ctx &C, const uint32_t n, uint32_t &max_nseg, uint32_t &min_nseg,
                                            uint32_t &np)
{
    const uint32_t maxn = __reduce_max_sync(0xFFFFFFFFu, n);
    max_nseg = (maxn + 7u) >> 3;
    min_nseg = __reduce_min_sync(0xFFFFFFFFu, (n + 7u) >> 3);
    np = C.pads_ok && max_nseg > 0 ? (maxn - 8u * (max_nseg - 1u)) >> 1 : 4u;
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

// y is read once and y' written once per SpMV: stream them past L2
// (evict-first loads, .cs stores) so the gathered x stays resident.
#ifndef DTANS_YSTREAM
#define DTANS_YSTREAM 1
#endif
#ifndef DTANS_YCS
#define DTANS_YCS 1
#endif
template <typename V> __device__ __forceinline__ V ld_stream(const V *p)
{
#if DTANS_YSTREAM && DTANS_YCS
    return __ldcs(p);  // ld.global.cs: evict-first in L1 and L2, no policy register
#elif DTANS_YSTREAM
    V v;
    if (sizeof(V) == 8) {
        unsigned long long b;
        asm("{\n.reg .b64 pol;\ncreatepolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
            "ld.global.nc.L1::no_allocate.L2::cache_hint.b64 %0, [%1], pol;\n}" : "=l"(b) : "l"(p));
        memcpy(&v, &b, 8);
    } else {
        uint32_t b;
        asm("{\n.reg .b64 pol;\ncreatepolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
            "ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], pol;\n}" : "=r"(b) : "l"(p));
        memcpy(&v, &b, 4);
    }
    return v;
#else
    return __ldg(p);
#endif
}
template <typename V> __device__ __forceinline__ void st_stream(V *p, V v)
{
#if DTANS_YSTREAM
    __stcs(p, v);
#else
    *p = v;
#endif
}

// consumption check (container.py:499-500) and column bound, one vote
// The same checks folded into a per-lane bit set (bit 0: consumption, bit 1:
// column bound), voted once per chunk (flush_bad) instead of once per slice.
__device__ __forceinline__ uint32_t bad_bits(const Ctx &C, bool ok, uint32_t cur, uint32_t end, uint32_t n,
                                             uint32_t col)
{
    return (!ok || cur != end ? 1u : 0u) | (n > 0 && col > C.cols_m1 ? 2u : 0u);
}
__device__ __forceinline__ void flush_bad(const KernelArgs &a, uint32_t &bad, int lane)
{
    if (__any_sync(0xFFFFFFFFu, bad != 0u)) {  // rare
        const uint32_t all = __reduce_or_sync(0xFFFFFFFFu, bad);
        if (lane == 0) atomicOr(a.err, all);
    }
    bad = 0u;
}

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

// One slice of a staged chunk: y (or decode positions) from global memory,
// everything else from shared memory.
template <typename V, bool kDecode, bool kHasY, bool kDIn, bool kScaled, bool kPend>
__device__ __forceinline__ void decode_slice(const KernelArgs &a, const Ctx &C, const V *__restrict__ x,
                                             SmemSrc src, const uint32_t end, const uint32_t meta,
                                             const uint32_t n, const uint32_t row, const int lane, const V scale,
                                             double &wsum, uint32_t &bad)
{
    using T = ValueTraits<V>;
    const bool inrow = row < (uint32_t)a.rows;
    const uint32_t max_nseg = (meta >> 16) & 0x7Fu;
    const uint32_t min_nseg = (meta >> 23) & 0x7Fu;
    const uint32_t np = (meta >> 30) + 1u;
    uint32_t orow = row;
    // the pending-products instantiation never runs with a row map (api.cu)
    if (!kPend && a.row_map != nullptr && inrow) orow = __ldg(a.row_map + row);
    V yv = V(0);
    if (kHasY && inrow) yv = ld_stream(reinterpret_cast<const V *>(a.y) + orow);
    LaneState<V> st;
    st.out_pos = 0;
    st.cur = 0;
    st.col = 0;
    st.acc = V(0);
    bool ok = true;
    if (max_nseg != 0u) {  // uniform; an all-empty slice has no words (y' = +0.0 + y)
        if (kDecode && inrow) st.out_pos = __ldg(a.row_start + row);
        init_state<V>(C, src, n, st);
#if DTANS_PEND2
        if (kPend && !kDecode && (meta & 0xFFFF0000u) == ((2u << 16) | (2u << 23))) {
            // uniform; the pending-products slice shape every 5-point
            // Laplacian slice has: two segments in every row, a one-pair final
            // segment (max_nseg = min_nseg = 2, np = 1) -- decode_range's pend
            // branch without its loop bookkeeping
            Pend4<V> pd;
            full_segment<V, kDecode, true, kDIn, SmemSrc, true>(a, C, x, src, 0u, n, 2u, st.w0, st.w1, st.w2, st.d,
                                                                 st.r, st.cur, st.col, st.acc, st.out_pos, lane, &pd);
            ok = st.cur <= end;
            if (ok) final_segment<V, kDecode, kDIn, 1, SmemSrc, true>(a, C, x, src, 1u, n, st, &pd);
        } else
#endif
            ok = decode_range<V, kDecode, kDIn, SmemSrc, kPend>(a, C, x, src, end, n, max_nseg, min_nseg, np, 0u,
                                                                max_nseg, st, lane);
    }
    bad |= bad_bits(C, ok, st.cur, end, n, st.col);
    if (!kDecode && inrow) {
        V res = kHasY ? T::add(st.acc, yv) : st.acc;
        if (kScaled) {
            // power iteration: y_k = (A y_{k-1}) / ||y_{k-1}||, sum of y_k^2
            res = T::mul(res, scale);
            wsum = __dadd_rn(wsum, __dmul_rn((double)res, (double)res));
        }
        st_stream(reinterpret_cast<V *>(a.out) + orow, res);
    }
}

__device__ __forceinline__ void st_shared_v2(uint32_t addr, uint32_t x, uint32_t y)
{
    asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(addr), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t x, uint32_t y, uint32_t z, uint32_t w)
{
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
__device__ __forceinline__ uint4 ld_shared_v4(uint32_t addr)
{
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ uint2 ld_shared_v2(uint32_t addr)
{
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr) : "memory");
    return v;
}

// Chunk staging (lane 0): one cp.async.bulk of the chunk's blob completing
// on the buffer's mbarrier.  The previous contents were consumed by this
// warp's LDS before the __syncwarp that precedes the call (the same WAR
// ordering a CUTLASS TMA pipeline relies on), so no proxy fence is issued.
// All addresses are shared-window addresses.
__device__ __forceinline__ void stage_chunk(const KernelArgs &a, const bool valid, const ChunkRec rc,
                                            const uint32_t bar, const uint32_t meta, const uint32_t buf)
{
    if (!valid) {
        st_shared_v2(meta, 0u, 0u);
        mbar_arrive(bar);
        return;
    }
    const uint32_t bytes = (rc.kw >> 8) * 4u;
    st_shared_v2(meta, rc.s0, rc.kw & 0xFFu);
    mbar_arrive_expect_tx(bar, bytes);
    bulk_g2s_stream(buf, a.blob + rc.off, bytes, bar);
}

// Per-warp control block of lane 0's claim pipeline (shared memory, so the
// other 31 lanes do not carry it in registers): the record of the next
// chunk to stage and the ticket of the one after.
struct WarpCtl {
    ChunkRec pend;
    uint32_t pend_c, next_static, pend_ok, pad;
    uint32_t hdr, rs, st, s0;  // the chunk being decoded (shared addresses), re-read per slice
    uint32_t cidx[kMaxRing], pad2[4 - kMaxRing];  // embedded records: chunk index staged in each buffer
};

// Persistent kernel, one CTA of 32 warps per SM: tables -> shared memory once,
// then every warp walks chunks (static stride or atomic tickets) through its
// TMA ring.
// kPend: decode_range may defer the last hot segment's products past a
// short final segment's gathers (a separate instantiation, chosen at upload
// for matrices where most slices take that path: it costs registers).  It is
// never launched with a row map, so it drops the row-map lookup.
template <typename V, bool kDecode, bool kHasY, bool kDIn, bool kScaled = false, bool kPend = false>
__global__ void __launch_bounds__(kMaxWarps * 32, 1) dtans_kernel(const KernelArgs a)
{
    // warps that decode: kMaxWarps, fewer for small matrices (api.cu); the
    // whole CTA still copies the tables in
    const uint32_t kWarps = (uint32_t)a.work_warps;
    pdl_trigger();
    const bool aligned = load_tables(a);
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const uint32_t sb = smem_u32(dtans_smem);
    const uint32_t bars = sb + (uint32_t)a.off_bars + (uint32_t)warp * kMaxRing * 8u;
    const uint32_t metas = sb + (uint32_t)a.off_meta + (uint32_t)warp * kMaxRing * 8u;
    WarpCtl *ctl = reinterpret_cast<WarpCtl *>(dtans_smem + a.off_ctl) + warp;
    if (lane == 0) {
        for (int b = 0; b < kMaxRing; b++) mbar_init(bars + 8u * b, 1);
        fence_mbar_init();
    }
    __syncthreads();
    // launched with PDL after the previous product's main kernel (api.cu
    // pdl_main): the table copy above overlapped its tail; x, y, the output
    // and the sums of squares are touched only after it has completed
    pdl_wait();
    if (!aligned) {  // shared-window layout assumption broken: fail loudly
        if (threadIdx.x == 0) atomicOr(a.err, 4u);
        return;
    }
    if (kScaled && a.sumsq_zero != nullptr && blockIdx.x == 0 && threadIdx.x == 0) *a.sumsq_zero = 0.0;
    if ((uint32_t)warp >= kWarps) return;  // helped with the table copy only
    const Ctx C = make_ctx<V>(a, lane);
    const V *__restrict__ x = reinterpret_cast<const V *>(a.x);
    V scale = V(1);
    double wsum = 0.0;
    if (kScaled) {
        if (a.sumsq_in != nullptr) {
            const double q = *a.sumsq_in;
            scale = (V)__ddiv_rn(1.0, __dsqrt_rn(q));
        }
    }

    // lane 0's claim pipeline.  Static plans built for this grid read the
    // next chunk record from the blob just decoded (embedded, no global
    // load); otherwise: ticket -> chunk record -> staged buffer.
    const uint32_t G = gridDim.x * kWarps;
    const bool emb = a.embed_stride == G && !a.dynamic;  // uniform
    auto claim = [&]() -> uint32_t {  // lane 0 only; >= chunk_hi: none
        if (a.dynamic) return a.chunk_lo + atomicAdd(a.work_counter, 1u);
        const uint32_t c = ctl->next_static;
        ctl->next_static = c + G;
        return c;
    };
    const uint32_t ctl_sh = sb + (uint32_t)a.off_ctl + (uint32_t)warp * (uint32_t)sizeof(WarpCtl);
    const uint32_t bufs = sb + (uint32_t)a.off_bufs + (uint32_t)warp * (uint32_t)(kMaxRing * a.bufb);
    if (lane == 0) {
        ctl->next_static = a.chunk_lo + blockIdx.x * kWarps + warp;
        for (int b = 0; b < kMaxRing; b++) {
            const uint32_t c = claim();
            const bool v = c < a.chunk_hi;
            ChunkRec rc{};
            if (v) rc = a.chunks[c];
            ctl->cidx[b] = c;
            stage_chunk(a, v, rc, bars + 8u * b, metas + 8u * b, bufs + b * (uint32_t)a.bufb);
        }
        if (!emb) {
            const uint32_t c = claim();
            ctl->pend_ok = c < a.chunk_hi;
            if (c < a.chunk_hi) ctl->pend = a.chunks[c];
            ctl->pend_c = claim();
        }
    }
    __syncwarp();
    uint32_t bad = 0u;  // this chunk's failed checks (bad_bits)
    for (uint32_t it = 0;; it++) {
        const uint32_t b = it & (kMaxRing - 1u);
        mbar_wait(bars + 8u * b, (it / kMaxRing) & 1u);
        const uint2 md = ld_shared_v2(metas + 8u * b);
        const uint32_t s0 = md.x, k = md.y;
        if (k == 0) break;  // uniform: this warp's chunks are exhausted
        // the chunk's addresses live in the warp's control block and are
        // re-read per slice (one LDS.128) instead of occupying registers
        // across the decode
        const uint32_t ctl_cs = ctl_sh + 32u;
        if (lane == 0) {
            const uint32_t buf = bufs + b * (uint32_t)a.bufb;
            const uint32_t hw = chunk_hdr_words(k);
            st_shared_v4(ctl_cs, buf + 16u, buf + hw * 4u, buf + (hw + k * 32u) * 4u, s0);
        }
        __syncwarp();
        uint32_t dcur = 0;
        for (uint32_t i = 0; i < k; i++) {
            const uint4 cs = ld_shared_v4(ctl_cs);
            const uint32_t meta = sh32(cs.x + 4u * i);
            const uint32_t dnext = meta & 0xFFFFu;
            const uint32_t n = sh32(cs.y + i * 128u + (uint32_t)lane * 4u);
            const SmemSrc src{cs.z + dcur * 4u};
            decode_slice<V, kDecode, kHasY, kDIn, kScaled, kPend>(a, C, x, src, dnext - dcur, meta, n,
                                                            (cs.w + i) * kSliceRows + (uint32_t)lane, lane, scale, wsum,
                                                            bad);
            dcur = dnext;
        }
        flush_bad(a, bad, lane);
        __syncwarp();
        if (lane == 0) {
            const uint32_t buf = bufs + b * (uint32_t)a.bufb;
            if (emb) {
                // the record of the chunk this buffer takes next, embedded in
                // the blob just decoded (read before the copy overwrites it)
                const uint32_t c = ctl->cidx[b] + kMaxRing * G;
                const bool v = c < a.chunk_hi;
                ChunkRec rc{};
                if (v) {
                    const uint4 r = ld_shared_v4(buf);
                    rc.off = (unsigned long long)r.x | (unsigned long long)r.y << 32;
                    rc.s0 = r.z;
                    rc.kw = r.w;
                }
                ctl->cidx[b] = c;
                stage_chunk(a, v, rc, bars + 8u * b, metas + 8u * b, buf);
            } else {
                stage_chunk(a, ctl->pend_ok != 0u, ctl->pend, bars + 8u * b, metas + 8u * b, buf);
                const uint32_t c = ctl->pend_c;
                ctl->pend_ok = c < a.chunk_hi;
                if (c < a.chunk_hi) ctl->pend = a.chunks[c];
                ctl->pend_c = claim();
            }
        }
        __syncwarp();
    }
    if (kScaled && a.sumsq_out != nullptr) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) wsum = __dadd_rn(wsum, __shfl_xor_sync(0xFFFFFFFFu, wsum, o));
        if (lane == 0) atomicAdd(a.sumsq_out, wsum);
    }
}

constexpr int kTaskWarps = DTANS_TASK_WARPS;  // task kernel CTA size (warps)

// Long-slice tasks: each warp decodes segments [j0, j1) of one slice from a
// checkpoint (or the init events), reading the stream from global memory
// (the task's words are prefetched into L1 first), and writes its 32
// per-lane partial sums (or, when decoding, the columns and value bits of
// those segments directly).  Staging the task words in shared memory instead
// (whole tasks, or a streamed window of cp.async.bulk quarters) measured
// slower: the shared-memory carve-out costs the x gathers their L1 (DESIGN 5c).
template <typename V, bool kDecode, bool kDIn>
__global__ void __launch_bounds__(kTaskWarps * 32, 1024 / (kTaskWarps * 32)) dtans_task_kernel(const KernelArgs a)
{
    pdl_trigger();
    const bool aligned = load_tables(a);
    __syncthreads();
    if (!aligned) {
        if (threadIdx.x == 0) atomicOr(a.err, 4u);
        pdl_wait();
        return;
    }
    const int lane = threadIdx.x & 31;
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t warps = blockDim.x >> 5;
    const Ctx C = make_ctx<V>(a, lane);
    const V *__restrict__ x = reinterpret_cast<const V *>(a.x);
#if DTANS_GMEM_CS == 0
    const unsigned long long pol = policy_evict_first();
#endif
    // power iteration (sumsq_out set): single-task slices are final here, so
    // they are scaled and their squares summed like the main kernel's rows
    const V scale = a.sumsq_in != nullptr ? (V)__ddiv_rn(1.0, __dsqrt_rn(*a.sumsq_in)) : V(1);
    double wsum = 0.0;
    const uint32_t tstride = gridDim.x * warps;
    // static tasks t, t + tstride, ...; or (a.task_dyn, when the kernel runs
    // beside the solo kernel and some CTAs start late) tickets past the
    // static first round from work_counter[1], zeroed per launch
    uint32_t t = blockIdx.x * warps + warp;
#if DTANS_TICKET_BATCH
    uint32_t tpend = 0xFFFFFFFFu;  // the second task of the claimed pair
#endif
    while (t < a.ntasks) {
        uint32_t tnext = t + tstride;
#if DTANS_TICKET_BATCH
        // one atomic per pair of tasks: ticket c -> tasks tstride + 2c and
        // tstride + 2c + 1 (the warp-aggregated atomic waits for its result
        // at once -- ptxas -- so half the claims halve those waits)
        if (a.task_dyn) {
            if (tpend != 0xFFFFFFFFu) {
                tnext = tpend;
                tpend = 0xFFFFFFFFu;
            } else {
                uint32_t c = 0;
                if (lane == 0) c = atomicAdd(a.work_counter + 1, 1u);
                tnext = tstride + 2u * __shfl_sync(0xFFFFFFFFu, c, 0);
                tpend = tnext + 1u;
            }
        }
#else
        if (a.task_dyn && lane == 0) tnext = tstride + atomicAdd(a.work_counter + 1, 1u);
#endif
        const LongTask tk = a.tasks[t];
        const uint32_t row = tk.slice * kSliceRows + lane;
        const bool inrow = row < (uint32_t)a.rows;
        const uint32_t n = inrow ? __ldg(a.row_symbols + row) : 0u;
        uint32_t max_nseg, min_nseg, np;
        slice_shape(C, n, max_nseg, min_nseg, np);
        // the task's words [cur0, cur1) of the slice (a first task also reads
        // the init words from 0); positions are task-relative
        const uint32_t w0 = tk.ck == 0xFFFFFFFFu ? 0u : tk.cur0;
        const uint64_t g0 = __ldg(a.directory + tk.slice) + w0;
        const uint32_t ntw = tk.cur1 - w0;
#if DTANS_GMEM_CS == 0
        GmemSrc src{a.stream + g0, pol};
#else
        GmemSrc src{a.stream + g0};
#endif
        {
            // pull the task's stream words into L1 up front (coalesced line
            // prefetches) so the loads on the serial per-segment chain hit L1
            const char *b = reinterpret_cast<const char *>(src.p);
            const char *e = reinterpret_cast<const char *>(src.p + ntw);
            for (const char *q = b + 128 * lane; q < e; q += 128 * 32) asm volatile("prefetch.global.L1 [%0];" ::"l"(q));
        }
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
            st.cur = 0u;
            st.acc = V(0);
        }
        // decoding: every segment before j0 of an active lane was full (4 pairs)
        if (kDecode && inrow) st.out_pos = __ldg(a.row_start + row) + 4ll * tk.j0;
        const bool ok = decode_range<V, kDecode, kDIn>(a, C, x, src, ntw, n, max_nseg, min_nseg, np, tk.j0, tk.j1,
                                                       st, lane);
        report(a, C, ok, st.cur, ntw, tk.last ? n : 0u, st.col, lane);
        if (!kDecode) {
            if (tk.last && tk.j0 == 0) {
                // the slice is this single task: y' = acc + y directly
                if (inrow) {
                    const uint32_t orow = a.row_map != nullptr ? __ldg(a.row_map + row) : row;
                    V res = st.acc;
                    if (a.y != nullptr) res = ValueTraits<V>::add(res, reinterpret_cast<const V *>(a.y)[orow]);
                    if (a.sumsq_out != nullptr) {
                        res = ValueTraits<V>::mul(res, scale);
                        wsum = __dadd_rn(wsum, __dmul_rn((double)res, (double)res));
                    }
                    reinterpret_cast<V *>(a.out)[orow] = res;
                }
            } else {
                reinterpret_cast<V *>(a.partials)[(size_t)tk.part * 32 + lane] = st.acc;
            }
        }
#if DTANS_TICKET_BATCH
        t = tnext;
#else
        t = a.task_dyn ? __shfl_sync(0xFFFFFFFFu, tnext, 0) : tnext;
#endif
    }
    if (!kDecode && a.sumsq_out != nullptr) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) wsum = __dadd_rn(wsum, __shfl_xor_sync(0xFFFFFFFFu, wsum, o));
        if (lane == 0 && wsum != 0.0) atomicAdd(a.sumsq_out, wsum);
    }
    pdl_wait();
}

// Solo tasks: one THREAD decodes segments [j0, j1) of the only row still
// active in its long slice.  With a single active lane every event of the
// slice belongs to that row (container.py:406-413 with one lane), so its
// words are consecutive from cur0 and the lockstep ballots reduce to a
// running cursor; 32 independent chunks share a warp.
template <typename V, bool kDecode, bool kDIn>
__global__ void __launch_bounds__(256) dtans_solo_kernel(const KernelArgs a)
{
    using T = ValueTraits<V>;
    using Bits = typename T::Bits;
    pdl_trigger();
    const bool aligned = load_tables(a);
    __syncthreads();
    if (!aligned) {
        if (threadIdx.x == 0) atomicOr(a.err, 4u);
        pdl_wait();
        return;
    }
    const Ctx C = make_ctx<V>(a, (int)(threadIdx.x & 31));
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
            slot_offsets(C.tab, w0, w1, w2, so);
#pragma unroll
            for (int p = 0; p < 4; p++)
                lookup_pair<Bits, kDIn>(C, so[2 * p], so[2 * p + 1], e[2 * p], e[2 * p + 1], ds[p], vs[p]);
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
    pdl_wait();
}

// Checkpoint walk (the GPU pre-pass of the long-slice index): one warp per
// long slice replays the lockstep decode (decode_range in decode mode with no
// output arrays) and, at every task boundary j = 0, chunk, 2 chunk, ..., of
// the host's plan (checkpoints.cpp build_long_index), records the slice
// cursor in cursors[part] and -- for j > 0 -- the resume record of the
// lanes still active: {mask, 6 words per lane} for a warp task, the lane's
// 6 words for a solo task (a single lane left), at the record offsets the
// host assigned in the same order.  The final cursor must equal the slice's
// word count.  WalkSrc hooks the per-segment prepare() of decode_range.
template <typename V> struct WalkSrc {
    const uint32_t *p;        // &stream[directory[s]]
    const LaneState<V> *st;   // the walking lanes' state (read at segment starts)
    uint32_t *pool;           // this slice's first resume record
    uint32_t *cursors;        // cursors[part_base + k]
    uint32_t n, chunk, j, k;  // lane's row symbols; segments per task; segment; boundary
    __device__ __forceinline__ uint32_t operator()(uint32_t rel) const { return __ldg(p + rel); }
    __device__ __forceinline__ void prepare(uint32_t cur)
    {
        if (j % chunk == 0u) {  // uniform
            const int lane = threadIdx.x & 31;
            if (lane == 0) cursors[k] = cur;
            if (j > 0u) {
                const uint32_t mask = __ballot_sync(0xFFFFFFFFu, ((n + 7u) >> 3) > j);
                const bool act = (mask >> lane) & 1u;
                const uint32_t rk = __popc(mask & lanemask_lt());
                uint32_t *rec = pool;
                if (__popc(mask) == 1u) {
                    pool += 6;
                } else {
                    if (lane == 0) rec[0] = mask;
                    rec += 1 + 6 * rk;
                    pool += 1 + 6 * __popc(mask);
                }
                if (act) {
                    rec[0] = st->w0;
                    rec[1] = st->w1;
                    rec[2] = st->w2;
                    rec[3] = st->d;
                    rec[4] = st->r;
                    rec[5] = st->col;
                }
            }
            k++;
        }
        j++;
    }
};

template <typename V, bool kDIn>
__global__ void __launch_bounds__(256) dtans_walk_kernel(const KernelArgs a, uint32_t *pool, uint32_t *cursors,
                                                         uint32_t *final_cur, uint32_t chunk)
{
    const bool aligned = load_tables(a);
    __syncthreads();
    if (!aligned) {
        if (threadIdx.x == 0) atomicOr(a.err, 4u);
        return;
    }
    const int lane = threadIdx.x & 31;
    const Ctx C = make_ctx<V>(a, lane);
    const uint32_t warps = blockDim.x >> 5;
    for (uint32_t i = blockIdx.x * warps + (threadIdx.x >> 5); i < a.nlong; i += gridDim.x * warps) {
        const LongSlice ls = a.longs[i];
        const uint32_t row = ls.slice * kSliceRows + lane;
        const uint32_t n = row < (uint32_t)a.rows ? __ldg(a.row_symbols + row) : 0u;
        uint32_t max_nseg, min_nseg, np;
        slice_shape(C, n, max_nseg, min_nseg, np);
        const uint64_t d0 = __ldg(a.directory + ls.slice);
        const uint32_t nw = (uint32_t)(__ldg(a.directory + ls.slice + 1) - d0);
        LaneState<V> st;
        st.out_pos = 0;
        WalkSrc<V> src{a.stream + d0, &st, pool + ls.pool_base, cursors + ls.part_base, n, chunk, 0u, 0u};
        init_state<V>(C, src, n, st);
        const bool ok = decode_range<V, true, kDIn>(a, C, nullptr, src, nw, n, max_nseg, min_nseg, np, 0u, max_nseg,
                                                    st, lane);
        if (lane == 0) final_cur[i] = ok ? st.cur : 0xFFFFFFFFu;
    }
}

// All-empty slices (every row has no symbols, no stream words) of a plan
// with long slices: y' = +0.0 + y per row (container.py:534-551 with an
// empty row), scaled like the main kernel's rows in a power iteration.
// Taken out of the chunk list because a staged chunk pays its per-slice
// chain (row map -> y -> y') one slice at a time; here each warp keeps four
// slices' loads in flight (a rows-sorted R-MAT: 142k empty slices).
template <typename V, bool kHasY>
__global__ void __launch_bounds__(256) dtans_empty_kernel(const KernelArgs a)
{
    using T = ValueTraits<V>;
    constexpr int kU = DTANS_EMPTY_UNROLL;
    pdl_trigger();
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const V scale = a.sumsq_in != nullptr ? (V)__ddiv_rn(1.0, __dsqrt_rn(*a.sumsq_in)) : V(1);
    const V *y = reinterpret_cast<const V *>(a.y);
    V *out = reinterpret_cast<V *>(a.out);
    double wsum = 0.0;
    for (uint32_t i0 = gw; i0 < a.nempty; i0 += kU * nw) {
        uint32_t orow[kU];
        bool in[kU];
#pragma unroll
        for (int u = 0; u < kU; u++) {
            const uint32_t i = i0 + (uint32_t)u * nw;
            const uint32_t row = i < a.nempty ? __ldg(a.empty_slices + i) * kSliceRows + lane : 0xFFFFFFFFu;
            in[u] = row < (uint32_t)a.rows;
            orow[u] = row;
        }
#pragma unroll
        for (int u = 0; u < kU; u++)
            if (in[u] && a.row_map != nullptr) orow[u] = __ldg(a.row_map + orow[u]);
        V res[kU];
#pragma unroll
        for (int u = 0; u < kU; u++) {
            res[u] = V(0);
            if (kHasY && in[u]) res[u] = T::add(V(0), ld_stream(y + orow[u]));
        }
#pragma unroll
        for (int u = 0; u < kU; u++) {
            if (!in[u]) continue;
            V r = res[u];
            if (a.sumsq_out != nullptr) {
                r = T::mul(r, scale);
                wsum = __dadd_rn(wsum, __dmul_rn((double)r, (double)r));
            }
            st_stream(out + orow[u], r);
        }
    }
    if (a.sumsq_out != nullptr) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) wsum = __dadd_rn(wsum, __shfl_xor_sync(0xFFFFFFFFu, wsum, o));
        if (lane == 0 && wsum != 0.0) atomicAdd(a.sumsq_out, wsum);
    }
    pdl_wait();
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
    pdl_wait();  // the task and solo kernels' partials
    // power iteration (sumsq_out set): scale, and sum the squares (one f64
    // atomic per warp)
    auto finish = [&](const LongSlice &ls, V s) {
        const uint32_t row = ls.slice * kSliceRows + lane;
        double sq = 0.0;
        if (row < (uint32_t)a.rows) {
            const uint32_t orow = a.row_map != nullptr ? __ldg(a.row_map + row) : row;
            if (kHasY) s = T::add(s, reinterpret_cast<const V *>(a.y)[orow]);
            if (a.sumsq_out != nullptr) {
                if (a.sumsq_in != nullptr) s = T::mul(s, (V)__ddiv_rn(1.0, __dsqrt_rn(*a.sumsq_in)));
                sq = __dmul_rn((double)s, (double)s);
            }
            reinterpret_cast<V *>(a.out)[orow] = s;
        }
        if (a.sumsq_out != nullptr) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sq = __dadd_rn(sq, __shfl_xor_sync(0xFFFFFFFFu, sq, o));
            if (lane == 0 && sq != 0.0) atomicAdd(a.sumsq_out, sq);
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

}  // namespace dev
}  // namespace dtans
