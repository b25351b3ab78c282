// Fused dtANS decode + SpMV for sm_100a.
//
// One warp decodes one 32-row slice, lane i = row 32s+i, exactly the
// lockstep the container's word order was interleaved for
// (container.py:211-335).  Per lane the decoder runs the reference's
// per-segment loop (container.py:370-521, codec.py:384-453):
//   unpack 3 words -> 8 slots, 8 table lookups (shared memory),
//   escape payload event (warp exclusive scan), 2 mixed-radix checks
//   (extract from the state or load: ballot + popc), 1 unconditional load.
// The symbols never leave registers: column deltas are prefix-summed,
// x[col] is gathered and acc = fl(acc + fl(v * x)) runs left to right per
// row from +0.0 (container.py:534-551) with __dmul_rn/__dadd_rn, so the
// result is bitwise the reference's.
//
// Mixed-radix state: at every segment start d < r < 2^32 (r is divided by
// 2^32 whenever it reaches 2^32), so the resting state is two u32.  A group
// of 4 digits is folded into one product in 32-bit arithmetic using the
// decremented radix Bm1 = b0 b1 b2 b3 - 1 <= 2^32 - 1 (codec.py:127-137):
//   d' = d*Bm1 + d + D,  r' = r*Bm1 + r       (64-bit, < 2^64)
// and the check is r' >= 2^32: extract w = lo32(d'), d = hi32(d'),
// r = hi32(r'); else load (d', r' already fit 32 bits).
#pragma once
#include <cstdint>

namespace dtans {
namespace dev {

constexpr int kSliceRows = 32;
constexpr int kSlots = 4096;

// Slot-table entry layouts in shared memory (built by dtans_upload):
//   delta       : uint2 {sym32, meta}
//   value (f64) : uint4 {sym_lo, sym_hi, meta, 0}
//   value (f32) : uint2 {sym32, meta}
// meta = digit | (base-1) << 8 | escape << 16.
template <typename V> struct ValueTraits;
template <> struct ValueTraits<double> {
    using Entry = uint4;
    using Bits = unsigned long long;
    static constexpr int kPayloadWords = 2;
    __device__ static inline Bits sym(const uint4 &e)
    {
        return ((Bits)e.y << 32) | e.x;
    }
    __device__ static inline uint32_t meta(const uint4 &e) { return e.z; }
    __device__ static inline double from_bits(Bits b) { return __longlong_as_double((long long)b); }
    __device__ static inline double mul(double a, double b) { return __dmul_rn(a, b); }
    __device__ static inline double add(double a, double b) { return __dadd_rn(a, b); }
};
template <> struct ValueTraits<float> {
    using Entry = uint2;
    using Bits = uint32_t;
    static constexpr int kPayloadWords = 1;
    __device__ static inline Bits sym(const uint2 &e) { return e.x; }
    __device__ static inline uint32_t meta(const uint2 &e) { return e.y; }
    __device__ static inline float from_bits(Bits b) { return __uint_as_float(b); }
    __device__ static inline float mul(float a, float b) { return __fmul_rn(a, b); }
    __device__ static inline float add(float a, float b) { return __fadd_rn(a, b); }
};

struct KernelArgs {
    const uint2 *dtab;            // delta table (global copy)
    const void *vtab;             // value table (global copy)
    const uint32_t *row_symbols;  // rows
    const uint64_t *directory;    // nslices + 1
    const uint32_t *stream;       // nwords (+ padding)
    int64_t rows, cols, nslices, nwords;
    const void *x;
    const void *y;                // may be null
    void *out;
    const int64_t *row_start;     // decode kernel only
    int64_t *dec_cols;            // decode kernel only
    void *dec_vals;               // decode kernel only
    unsigned int *err;            // bit 0: consumption mismatch, bit 1: column OOB
    int decode_only;
};

__device__ __forceinline__ uint32_t lanemask_lt()
{
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ uint32_t ld_stream(const uint32_t *s, uint64_t pos)
{
    return __ldg(s + pos);
}

template <typename V>
__device__ __forceinline__ void decode_slice(const KernelArgs &a, const uint2 *__restrict__ sd,
                                             const typename ValueTraits<V>::Entry *__restrict__ sv,
                                             int64_t s, int lane)
{
    using T = ValueTraits<V>;
    using Bits = typename T::Bits;
    const uint32_t FULL = 0xFFFFFFFFu;
    const int64_t row = s * kSliceRows + lane;
    const bool inrow = row < a.rows;
    const uint32_t n = inrow ? __ldg(a.row_symbols + row) : 0u;
    const uint32_t nseg = (n + 7u) >> 3;
    const uint32_t max_nseg = __reduce_max_sync(FULL, nseg);
    uint64_t cur = __ldg(a.directory + s);
    const uint64_t end = __ldg(a.directory + s + 1);
    const uint64_t last_word = a.nwords > 0 ? (uint64_t)(a.nwords - 1) : 0;
    const uint32_t lt = lanemask_lt();
    const uint32_t *__restrict__ st = a.stream;

    // init events: 3 words per active lane
    uint32_t w0 = 0, w1 = 0, w2 = 0;
    {
        const uint32_t am = __ballot_sync(FULL, nseg > 0);
        const uint32_t cnt = __popc(am), rk = __popc(am & lt);
        if (nseg > 0) {
            w0 = ld_stream(st, min(cur + rk, last_word));
            w1 = ld_stream(st, min(cur + cnt + rk, last_word));
            w2 = ld_stream(st, min(cur + 2 * cnt + rk, last_word));
        }
        cur += 3 * cnt;
    }
    uint32_t d = 0, r = 1;
    uint32_t col = 0;
    bool col_bad = false;
    V acc = V(0);
    int64_t out_pos = 0;
    if (a.decode_only && inrow) out_pos = a.row_start[row];

    for (uint32_t j = 0; j < max_nseg; j++) {
        const bool act = j < nseg;
        const bool notlast = j + 1 < nseg;
        // unpack (codec.py:148-162): slot k = bits [12k, 12k+12) of w0:w1:w2
        uint32_t sl[8];
        sl[0] = w2 & 0xFFFu;
        sl[1] = (w2 >> 12) & 0xFFFu;
        sl[2] = __funnelshift_r(w2, w1, 24) & 0xFFFu;
        sl[3] = (w1 >> 4) & 0xFFFu;
        sl[4] = (w1 >> 16) & 0xFFFu;
        sl[5] = __funnelshift_r(w1, w0, 28) & 0xFFFu;
        sl[6] = (w0 >> 8) & 0xFFFu;
        sl[7] = w0 >> 20;
        uint2 de[4];
        typename T::Entry ve[4];
#pragma unroll
        for (int p = 0; p < 4; p++) {
            de[p] = sd[sl[2 * p]];
            ve[p] = sv[sl[2 * p + 1]];
        }
        uint32_t dsym[4];
        Bits vsym[4];
        uint32_t dmeta[4], vmeta[4];
        uint32_t pc = 0;
#pragma unroll
        for (int p = 0; p < 4; p++) {
            dsym[p] = de[p].x;
            dmeta[p] = de[p].y;
            vsym[p] = T::sym(ve[p]);
            vmeta[p] = T::meta(ve[p]);
            pc += (dmeta[p] >> 16) & 1u;
            pc += ((vmeta[p] >> 16) & 1u) * T::kPayloadWords;
        }
        if (!act) pc = 0;
        // payload event (container.py:459-470): exclusive scan of counts
        if (__any_sync(FULL, pc != 0)) {
            uint32_t incl = pc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += v;
            }
            const uint32_t total = __shfl_sync(FULL, incl, 31);
            uint64_t off = cur + (incl - pc);
            if (pc) {
#pragma unroll
                for (int p = 0; p < 4; p++) {
                    if ((dmeta[p] >> 16) & 1u) {
                        dsym[p] = ld_stream(st, min(off, last_word));
                        off += 1;
                    }
                    if ((vmeta[p] >> 16) & 1u) {
                        if (T::kPayloadWords == 2) {
                            const uint32_t lo = ld_stream(st, min(off, last_word));
                            const uint32_t hi = ld_stream(st, min(off + 1, last_word));
                            vsym[p] = (Bits)(((unsigned long long)hi << 32) | lo);
                        } else {
                            vsym[p] = (Bits)ld_stream(st, min(off, last_word));
                        }
                        off += T::kPayloadWords;
                    }
                }
            }
            cur += total;
        }
        // mixed-radix checks: bases only decide load vs extract
        uint32_t bm1g[2], dg[2];
#pragma unroll
        for (int g = 0; g < 2; g++) {
            // positions 4g..4g+3: delta, value, delta, value
            const uint32_t m0 = dmeta[2 * g], m1 = vmeta[2 * g];
            const uint32_t m2 = dmeta[2 * g + 1], m3 = vmeta[2 * g + 1];
            const uint32_t b0 = ((m0 >> 8) & 0xFFu) + 1u, b1 = ((m1 >> 8) & 0xFFu) + 1u;
            const uint32_t b2 = ((m2 >> 8) & 0xFFu) + 1u, b3m1 = (m3 >> 8) & 0xFFu;
            const uint32_t P = b0 * b1 * b2;                      // <= 2^24
            bm1g[g] = P * b3m1 + (P - 1u);                         // b0 b1 b2 b3 - 1
            dg[g] = (((m0 & 0xFFu) * b1 + (m1 & 0xFFu)) * b2 + (m2 & 0xFFu)) * (b3m1 + 1u) +
                    (m3 & 0xFFu);
        }
        // radix chain (depends on bases only) -> load flags of both checks
        const unsigned long long r1 = (unsigned long long)r * bm1g[0] + r;
        const bool ext0 = (r1 >> 32) != 0;
        const uint32_t ra = ext0 ? (uint32_t)(r1 >> 32) : (uint32_t)r1;
        const unsigned long long r2 = (unsigned long long)ra * bm1g[1] + ra;
        const bool ext1 = (r2 >> 32) != 0;
        const bool ld0 = notlast && !ext0, ld1 = notlast && !ext1;
        const uint32_t m_ld0 = __ballot_sync(FULL, ld0);
        const uint32_t m_ld1 = __ballot_sync(FULL, ld1);
        const uint32_t m_nl = __ballot_sync(FULL, notlast);
        const uint64_t p0 = cur + __popc(m_ld0 & lt);
        const uint64_t c1 = cur + __popc(m_ld0);
        const uint64_t p1 = c1 + __popc(m_ld1 & lt);
        const uint64_t c2 = c1 + __popc(m_ld1);
        const uint64_t p2 = c2 + __popc(m_nl & lt);
        cur = c2 + __popc(m_nl);
        uint32_t lw0 = 0, lw1 = 0, lw2 = 0;
        if (ld0) lw0 = ld_stream(st, min(p0, last_word));
        if (ld1) lw1 = ld_stream(st, min(p1, last_word));
        if (notlast) lw2 = ld_stream(st, min(p2, last_word));

        // symbols of this segment -> columns, values, products
#pragma unroll
        for (int p = 0; p < 4; p++) {
            const bool valid = act && (8u * j + 2u * p) < n;
            if (valid) {
                col += dsym[p];
                const bool oob = col >= (uint64_t)a.cols;
                col_bad |= oob;
                const uint32_t c = oob ? 0u : col;
                if (a.decode_only) {
                    a.dec_cols[out_pos] = (int64_t)col;
                    reinterpret_cast<Bits *>(a.dec_vals)[out_pos] = vsym[p];
                    out_pos++;
                } else {
                    const V xv = __ldg(reinterpret_cast<const V *>(a.x) + c);
                    acc = T::add(acc, T::mul(T::from_bits(vsym[p]), xv));
                }
            }
        }
        // digit chain
        if (notlast) {
            const unsigned long long d1 =
                (unsigned long long)d * bm1g[0] + ((unsigned long long)d + dg[0]);
            uint32_t da;
            if (ext0) {
                w0 = (uint32_t)d1;
                da = (uint32_t)(d1 >> 32);
            } else {
                w0 = lw0;
                da = (uint32_t)d1;
            }
            const unsigned long long d2 =
                (unsigned long long)da * bm1g[1] + ((unsigned long long)da + dg[1]);
            if (ext1) {
                w1 = (uint32_t)d2;
                d = (uint32_t)(d2 >> 32);
                r = (uint32_t)(r2 >> 32);
            } else {
                w1 = lw1;
                d = (uint32_t)d2;
                r = (uint32_t)r2;
            }
            w2 = lw2;
        }
    }
    if (lane == 0 && cur != end) atomicOr(a.err, 1u);
    if (__any_sync(FULL, col_bad) && lane == 0) atomicOr(a.err, 2u);
    if (!a.decode_only && inrow) {
        V res = acc;
        if (a.y) res = T::add(acc, reinterpret_cast<const V *>(a.y)[row]);
        reinterpret_cast<V *>(a.out)[row] = res;
    }
}

// Persistent kernel: tables -> shared memory once per CTA, then every warp
// walks slices with a grid-wide stride.
template <typename V>
__global__ void __launch_bounds__(512, 1) dtans_spmv_kernel(KernelArgs a)
{
    using Entry = typename ValueTraits<V>::Entry;
    extern __shared__ __align__(16) unsigned char smem[];
    uint2 *sd = reinterpret_cast<uint2 *>(smem);
    Entry *sv = reinterpret_cast<Entry *>(smem + kSlots * sizeof(uint2));
    {
        const int4 *src = reinterpret_cast<const int4 *>(a.dtab);
        int4 *dst = reinterpret_cast<int4 *>(sd);
        for (int i = threadIdx.x; i < kSlots * (int)sizeof(uint2) / 16; i += blockDim.x)
            dst[i] = __ldg(src + i);
        const int4 *vsrc = reinterpret_cast<const int4 *>(a.vtab);
        int4 *vdst = reinterpret_cast<int4 *>(sv);
        for (int i = threadIdx.x; i < kSlots * (int)sizeof(Entry) / 16; i += blockDim.x)
            vdst[i] = __ldg(vsrc + i);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int warps = blockDim.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * warps + (threadIdx.x >> 5);
    const int64_t stride = (int64_t)gridDim.x * warps;
    for (int64_t s = gw; s < a.nslices; s += stride) decode_slice<V>(a, sd, sv, s, lane);
}

}  // namespace dev
}  // namespace dtans
