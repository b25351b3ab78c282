// GPU encoder (sm_100a): encode_matrix (container.py:126-204) with its
// per-symbol passes on the device, byte-identical to the reference (and to
// the host encoder in encoder.cpp).
//
//   1. validation + symbol extraction (CsrMatrix.validate sparse.py:76-91,
//      matrix_deltas sparse.py:289-299, value_patterns sparse.py:302-309):
//      one thread per nonzero;
//   2. distributions (container.py:112-114, np.unique: ascending symbols with
//      counts): device radix sort + run-length encode (CUB);
//   3. quantize + build_tables (entropy.py:223-436) on the host: the one
//      floating-point step, shared with the host encoder (prepare_tables);
//   4. base pass (codec.py:278-293): one warp per slice, lane = row, writes
//      each segment's load flags and the slice's word count;
//   5. directory = exclusive scan of the slice word counts (CUB);
//   6. digit pass + interleave (codec.py:296-368, container.py:254-317): one
//      warp per slice walks the segments BACKWARD in lockstep.  The decoder's
//      event order per segment is payload, check 0, check 1, unconditional
//      (container.py:406-497), so walking the events backward from
//      directory[s+1] each lane's word lands at (event start + its rank among
//      the event's lanes), exactly where the forward interleave of the
//      reference puts it, while the lane runs the reference's backward digit
//      pass (un-extract, digit = d mod b, d //= b) in registers.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.h"
#include "encoder_internal.h"

namespace dtans {
namespace genc {

constexpr uint32_t FULL = 0xFFFFFFFFu;
constexpr unsigned kErrCoding = 1u, kErrCorrupt = 2u, kErrColRange = 4u, kErrColOrder = 8u, kErrRowStart = 16u;

struct DevDomain {
    const uint64_t *ret_sym;  // retained symbols, ascending (= id order)
    const uint16_t *id_base;  // base of each retained id
    const uint32_t *id_off;   // id -> first entry of slot_by_digit
    const uint16_t *slot_by_digit;
    const uint16_t *esc_slot;  // (ESCAPE, digit) -> slot, full-base escape run
    int32_t nret, esc_base, pad_id, has_pad, payload_words;
};

struct Args {
    int64_t rows, cols, nnz, nslices;
    int32_t prec;
    const int64_t *row_start;
    const int64_t *col;
    const void *vals;
    const uint8_t *head;  // 1 at the first nonzero of each row (extract pass)
    uint32_t *dkey;       // delta symbols (extract pass)
    void *vkey;           // value bit patterns (extract pass)
    DevDomain dom[2];
    uint8_t *flags;        // load flags of segment j of a row at row_start[row] + j
    uint64_t *slice_words; // base pass output
    const uint64_t *directory;
    uint32_t *stream;
    unsigned int *err;
};

__global__ void mark_heads(const Args a, uint8_t *head)
{
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < a.rows; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t lo = a.row_start[r], hi = a.row_start[r + 1];
        if (hi < lo) atomicOr(a.err, kErrRowStart);
        else if (hi > lo) head[lo] = 1;
    }
}

// matrix_deltas (sparse.py:289-299): delta_0 = col_0, delta_q = col_q - col_{q-1};
// value_patterns (sparse.py:302-309): the values' bit patterns.
template <typename VB>
__global__ void extract(const Args a)
{
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < a.nnz; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = a.col[q];
        if (c < 0 || c >= a.cols) atomicOr(a.err, kErrColRange);
        uint32_t dl = (uint32_t)c;
        if (!a.head[q]) {
            const int64_t p = a.col[q - 1];
            if (c <= p) atomicOr(a.err, kErrColOrder);
            dl = (uint32_t)(c - p);
        }
        a.dkey[q] = dl;
        reinterpret_cast<VB *>(a.vkey)[q] = reinterpret_cast<const VB *>(a.vals)[q];
    }
}

// Shared copies of both domains' retained-symbol lists (binary search keys).
struct SmemKeys {
    const uint64_t *rs[2];
};

__device__ __forceinline__ int32_t find_id(const uint64_t *rs, int32_t n, uint64_t key)
{
    int32_t lo = 0, hi = n;
    while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        if (rs[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return (lo < n && rs[lo] == key) ? lo : -1;
}

struct PosInfo {
    uint32_t base;
    int32_t id;        // retained id, -1 = escape
    uint64_t payload;  // escaped symbol
};

// Position t of a row (codec.py:241-263 _position_info): even = delta
// domain, odd = value domain; t >= n is a pad (entropy.py:392-401: the pad
// symbol, or an escape with payload 0 when the table is escape-only).
__device__ __forceinline__ PosInfo pos_info(const Args &a, const SmemKeys &K, int64_t lo, uint32_t n, uint32_t t)
{
    const int dom = t & 1;
    const DevDomain &D = a.dom[dom];
    PosInfo p;
    p.payload = 0;
    if (t >= n) {
        if (D.has_pad) {
            p.id = D.pad_id;
            p.base = __ldg(D.id_base + D.pad_id);
        } else {
            p.id = -1;
            p.base = (uint32_t)D.esc_base;
        }
    } else {
        const int64_t q = lo + (t >> 1);
        uint64_t sym;
        if (dom == 0) {
            const int64_t c = __ldg(a.col + q);
            sym = (uint64_t)(uint32_t)(t < 2 ? c : c - __ldg(a.col + q - 1));
        } else if (a.prec == 8) {
            sym = __ldg(reinterpret_cast<const unsigned long long *>(a.vals) + q);
        } else {
            sym = __ldg(reinterpret_cast<const uint32_t *>(a.vals) + q);
        }
        p.id = find_id(K.rs[dom], D.nret, sym);
        if (p.id >= 0) {
            p.base = __ldg(D.id_base + p.id);
        } else {
            p.base = (uint32_t)D.esc_base;
            p.payload = sym;
        }
    }
    if (p.base == 0) {  // not retained and no escape entry (codec.py:250-260)
        atomicOr(a.err, kErrCoding);
        p.base = 1;
    }
    return p;
}

__device__ __forceinline__ SmemKeys load_keys(const Args &a)
{
    extern __shared__ uint64_t keys[];
    for (int i = threadIdx.x; i < a.dom[0].nret; i += blockDim.x) keys[i] = a.dom[0].ret_sym[i];
    for (int i = threadIdx.x; i < a.dom[1].nret; i += blockDim.x) keys[a.dom[0].nret + i] = a.dom[1].ret_sym[i];
    __syncthreads();
    SmemKeys K;
    K.rs[0] = keys;
    K.rs[1] = keys + a.dom[0].nret;
    return K;
}

// Base pass (codec.py:278-293): the load flags follow from the bases alone;
// words per lane = init 3 + payloads + per non-final segment (loaded checks + 1).
__global__ void __launch_bounds__(256) base_pass(const Args a)
{
    const SmemKeys K = load_keys(a);
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t s = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); s < a.nslices; s += warps) {
        const int64_t row = s * kSlice + lane;
        int64_t lo = 0, nnz = 0;
        if (row < a.rows) {
            lo = a.row_start[row];
            nnz = a.row_start[row + 1] - lo;
        }
        const uint32_t n = (uint32_t)(2 * nnz);
        const uint32_t nseg = (n + 7u) >> 3;
        uint64_t words = n ? 3u : 0u, r = 1;
        for (uint32_t j = 0; j < nseg; j++) {
            uint32_t b[8];
#pragma unroll
            for (int k = 0; k < 8; k++) {
                const PosInfo p = pos_info(a, K, lo, n, 8u * j + k);
                b[k] = p.base;
                if (p.id < 0) words += (k & 1) ? (uint32_t)a.dom[1].payload_words : 1u;
            }
            if (j + 1 < nseg) {
                uint8_t f = 0;
#pragma unroll
                for (int c = 0; c < 2; c++) {
#pragma unroll
                    for (int k = 4 * c; k < 4 * c + 4; k++) r *= b[k];
                    if (r >> 32) r >>= 32;
                    else f |= (uint8_t)(1u << c);
                }
                a.flags[lo + j] = f;
                words += 1u + (f & 1u) + (f >> 1);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) words += __shfl_xor_sync(FULL, words, o);
        if (lane == 0) a.slice_words[s] = words;
    }
}

__device__ __forceinline__ uint16_t reverse_slot(const DevDomain &D, const PosInfo &p, uint32_t digit)
{
    if (p.id < 0) return __ldg(D.esc_slot + digit);
    return __ldg(D.slot_by_digit + __ldg(D.id_off + p.id) + digit);
}

// pack (codec.py:165-180): slot 0 least significant, w0 most significant.
__device__ __forceinline__ void pack(const uint16_t s[8], uint32_t &w0, uint32_t &w1, uint32_t &w2)
{
    w2 = (uint32_t)s[0] | (uint32_t)s[1] << 12 | (uint32_t)(s[2] & 0xFFu) << 24;
    w1 = (uint32_t)s[2] >> 8 | (uint32_t)s[3] << 4 | (uint32_t)s[4] << 16 | (uint32_t)(s[5] & 0xFu) << 28;
    w0 = (uint32_t)s[5] >> 4 | (uint32_t)s[6] << 8 | (uint32_t)s[7] << 20;
}

// Digit pass + interleave, one warp per slice walking the events backward.
__global__ void __launch_bounds__(256) emit_pass(const Args a)
{
    const SmemKeys K = load_keys(a);
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t s = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); s < a.nslices; s += warps) {
        const int64_t row = s * kSlice + lane;
        int64_t lo = 0, nnz = 0;
        if (row < a.rows) {
            lo = a.row_start[row];
            nnz = a.row_start[row + 1] - lo;
        }
        const uint32_t n = (uint32_t)(2 * nnz);
        const uint32_t nseg = (n + 7u) >> 3;
        const uint32_t max_nseg = __reduce_max_sync(FULL, nseg);
        uint64_t cur = a.directory[s + 1];
        uint64_t d = 0;
        uint32_t w0 = 0, w1 = 0, w2 = 0;  // packed slots of the segment after j
        for (int64_t jj = (int64_t)max_nseg - 1; jj >= 0; jj--) {
            const uint32_t j = (uint32_t)jj;
            const bool act = j < nseg, notlast = j + 1 < nseg;
            const uint32_t f = notlast ? a.flags[lo + j] : 0u;
            // unconditional load, then checks 1 and 0 (backward event order)
            uint32_t m = __ballot_sync(FULL, notlast);
            cur -= __popc(m);
            if (notlast) a.stream[cur + __popc(m & lt)] = w2;
            m = __ballot_sync(FULL, notlast && (f & 2u));
            cur -= __popc(m);
            if (notlast && (f & 2u)) a.stream[cur + __popc(m & lt)] = w1;
            m = __ballot_sync(FULL, notlast && (f & 1u));
            cur -= __popc(m);
            if (notlast && (f & 1u)) a.stream[cur + __popc(m & lt)] = w0;
            PosInfo p[8];
            uint16_t sl[8];
            uint32_t pc = 0;
            if (act) {
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    p[k] = pos_info(a, K, lo, n, 8u * j + k);
                    if (p[k].id < 0) pc += (k & 1) ? (uint32_t)a.dom[1].payload_words : 1u;
                }
                if (notlast) {
                    // codec.py:336-358: for c = 1, 0: un-extract unless loaded,
                    // then digits of the group's slots in reverse
#pragma unroll
                    for (int c = 1; c >= 0; c--) {
                        if (!(f & (1u << c))) d = (d << 32) | (c ? w1 : w0);
#pragma unroll
                        for (int k = 4 * c + 3; k >= 4 * c; k--) {
                            const uint64_t b = p[k].base;
                            const uint64_t qd = d / b;
                            sl[k] = reverse_slot(a.dom[k & 1], p[k], (uint32_t)(d - qd * b));
                            d = qd;
                        }
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < 8; k++) sl[k] = reverse_slot(a.dom[k & 1], p[k], 0u);
                }
            }
            // payload event: lanes in order, slots in order, low word first
            uint32_t incl = pc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += v;
            }
            const uint32_t tot = __shfl_sync(FULL, incl, 31);
            cur -= tot;
            if (act) {
                uint64_t off = cur + (incl - pc);
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    if (p[k].id >= 0) continue;
                    a.stream[off++] = (uint32_t)p[k].payload;
                    if ((k & 1) && a.dom[1].payload_words == 2) a.stream[off++] = (uint32_t)(p[k].payload >> 32);
                }
                pack(sl, w0, w1, w2);
            }
        }
        // init events c = 2, 1, 0 (backward)
        const uint32_t am = __ballot_sync(FULL, n > 0);
        const uint32_t cnt = __popc(am), rk = __popc(am & lt);
        cur -= cnt;
        if (n) a.stream[cur + rk] = w2;
        cur -= cnt;
        if (n) a.stream[cur + rk] = w1;
        cur -= cnt;
        if (n) a.stream[cur + rk] = w0;
        const bool bad = d != 0 || cur != a.directory[s];  // codec.py:364 / consumption
        if (__any_sync(FULL, bad) && lane == 0) atomicOr(a.err, kErrCorrupt);
    }
}

// Device buffers of one encode, freed on every exit path.  Stream-ordered
// allocations from the device's default memory pool, which keeps freed
// memory (release threshold raised once), so repeated encodes and the
// scratch of the sort do not pay cudaMalloc/cudaFree each time.
struct Buffers {
    std::vector<void *> ptrs;
    ~Buffers()
    {
        for (void *p : ptrs) cudaFreeAsync(p, 0);
    }
    template <typename T> cudaError_t alloc(T **p, size_t count)
    {
        void *q = nullptr;
        const cudaError_t e = cudaMallocAsync(&q, std::max<size_t>(count, 1) * sizeof(T), 0);
        if (e == cudaSuccess) ptrs.push_back(q);
        *p = (T *)q;
        return e;
    }
};

#define GK(call, what)                                                                   \
    do {                                                                                 \
        const cudaError_t e_ = (call);                                                   \
        if (e_ != cudaSuccess) {                                                         \
            dtans_encoded_free(out);                                                     \
            return fail(e_ == cudaErrorMemoryAllocation ? DTANS_E_NOMEM : DTANS_E_CUDA, \
                        "%s: %s", what, cudaGetErrorString(e_));                         \
        }                                                                                \
    } while (0)

// Sorted unique symbols with counts (np.unique) of n keys on the device.
template <typename KeyT>
int distribution(Buffers &B, const KeyT *keys, int64_t n, Dist &out_d, dtans_encoded *out)
{
    out_d = Dist();
    out_d.total = n;
    if (n == 0) return DTANS_OK;
    KeyT *sorted = nullptr, *uniq = nullptr;
    int64_t *counts = nullptr, *nruns = nullptr;
    GK(B.alloc(&sorted, n), "cudaMalloc");
    GK(B.alloc(&uniq, n), "cudaMalloc");
    GK(B.alloc(&counts, n), "cudaMalloc");
    GK(B.alloc(&nruns, 1), "cudaMalloc");
    size_t t1 = 0, t2 = 0;
    GK(cub::DeviceRadixSort::SortKeys(nullptr, t1, keys, sorted, n), "radix sort");
    GK(cub::DeviceRunLengthEncode::Encode(nullptr, t2, sorted, uniq, counts, nruns, n), "run-length encode");
    uint8_t *tmp = nullptr;
    GK(B.alloc(&tmp, std::max(t1, t2)), "cudaMalloc");
    GK(cub::DeviceRadixSort::SortKeys(tmp, t1, keys, sorted, n), "radix sort");
    GK(cub::DeviceRunLengthEncode::Encode(tmp, t2, sorted, uniq, counts, nruns, n), "run-length encode");
    int64_t nr = 0;
    GK(cudaMemcpy(&nr, nruns, sizeof(int64_t), cudaMemcpyDeviceToHost), "download");
    std::vector<KeyT> u((size_t)nr);
    out_d.cnt.resize((size_t)nr);
    GK(cudaMemcpy(u.data(), uniq, sizeof(KeyT) * (size_t)nr, cudaMemcpyDeviceToHost), "download");
    GK(cudaMemcpy(out_d.cnt.data(), counts, sizeof(int64_t) * (size_t)nr, cudaMemcpyDeviceToHost), "download");
    out_d.sym.assign(u.begin(), u.end());
    return DTANS_OK;
}

int upload_domain(Buffers &B, const Domain &D, DevDomain &dd, dtans_encoded *out)
{
    uint64_t *rs;
    uint16_t *ib, *sbd, *es;
    uint32_t *io;
    GK(B.alloc(&rs, D.ret_sym.size()), "cudaMalloc");
    GK(B.alloc(&ib, D.id_base.size()), "cudaMalloc");
    GK(B.alloc(&io, D.id_off.size()), "cudaMalloc");
    GK(B.alloc(&sbd, D.slot_by_digit.size()), "cudaMalloc");
    GK(B.alloc(&es, D.esc_slot.size()), "cudaMalloc");
    auto up = [](void *dst, const void *src, size_t bytes) {
        return bytes ? cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice) : cudaSuccess;
    };
    GK(up(rs, D.ret_sym.data(), 8 * D.ret_sym.size()), "upload");
    GK(up(ib, D.id_base.data(), 2 * D.id_base.size()), "upload");
    GK(up(io, D.id_off.data(), 4 * D.id_off.size()), "upload");
    GK(up(sbd, D.slot_by_digit.data(), 2 * D.slot_by_digit.size()), "upload");
    GK(up(es, D.esc_slot.data(), 2 * D.esc_slot.size()), "upload");
    dd.ret_sym = rs;
    dd.id_base = ib;
    dd.id_off = io;
    dd.slot_by_digit = sbd;
    dd.esc_slot = es;
    dd.nret = (int32_t)D.ret_sym.size();
    dd.esc_base = D.esc_base;
    dd.pad_id = D.pad_id;
    dd.has_pad = D.has_pad ? 1 : 0;
    dd.payload_words = D.payload_words;
    return DTANS_OK;
}

}  // namespace genc
}  // namespace dtans

using namespace dtans;
using namespace dtans::genc;

namespace {
// DTANS_VERBOSE: per-phase wall times of the GPU encoder.
struct PhaseTimer {
    bool on = getenv("DTANS_VERBOSE") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    char buf[512] = {0};
    size_t len = 0;
    void mark(const char *what)
    {
        if (!on) return;
        cudaDeviceSynchronize();
        const auto now = std::chrono::steady_clock::now();
        len += (size_t)snprintf(buf + len, sizeof(buf) - len, " %s %.3f", what,
                                std::chrono::duration<double>(now - t).count());
        t = now;
    }
    ~PhaseTimer()
    {
        if (on) fprintf(stderr, "[dtans] encode_device (s):%s\n", buf);
    }
};
}  // namespace

extern "C" int dtans_encode_device(const dtans_csr_view *m, const dtans_encode_opts *opts, int device,
                                   dtans_encoded *out)
{
    if (!m || !opts || !out) return fail(DTANS_E_PARAM, "null argument");
    memset(out, 0, sizeof(*out));
    const int prec = m->precision;
    if (prec != 4 && prec != 8) return fail(DTANS_E_PARAM, "precision must be 4 or 8 bytes");
    if (opts->k_log2 != kKLog2) return fail(DTANS_E_PARAM, "this build implements k = 4096");
    if (opts->m_log2 < 1 || opts->m_log2 > 8)
        return fail(DTANS_E_PARAM, "slot records store base - 1 in one byte; m <= 256");
    if (m->rows < 0 || m->cols < 0) return fail(DTANS_E_PARAM, "negative dimensions");
    if (m->cols > (int64_t)1 << 32 || m->rows > (int64_t)1 << 32)
        return fail(DTANS_E_PARAM, "indices must fit 32 bits");
    const int64_t rows = m->rows, nnz = m->nnz, nslices = (rows + kSlice - 1) / kSlice;
    if (nnz >= ((int64_t)1 << 31)) return fail(DTANS_E_PARAM, "the GPU encoder takes nnz < 2^31 (use dtans_encode)");
    if (m->row_start[0] != 0 || m->row_start[rows] != nnz) return fail(DTANS_E_PARAM, "row_start must span [0, nnz]");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(DTANS_E_NODEVICE, "no CUDA device visible: the GPU encoder needs one");
    }
    if (device < 0 || device >= ndev) return fail(DTANS_E_PARAM, "bad device ordinal %d", device);
    GK(cudaSetDevice(device), "cudaSetDevice");
    int sms = 0;
    GK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device), "sm count");
    {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t keep = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    }
    PhaseTimer pt;
    Buffers B;
    Args a{};
    a.rows = rows;
    a.cols = m->cols;
    a.nnz = nnz;
    a.nslices = nslices;
    a.prec = prec;
    int64_t *rs, *col;
    uint8_t *vals, *head;
    unsigned int *err;
    GK(B.alloc(&rs, rows + 1), "cudaMalloc");
    GK(B.alloc(&col, nnz), "cudaMalloc");
    GK(B.alloc(&vals, (size_t)nnz * prec), "cudaMalloc");
    GK(B.alloc(&head, nnz), "cudaMalloc");
    GK(B.alloc(&err, 1), "cudaMalloc");
    GK(cudaMemcpy(rs, m->row_start, sizeof(int64_t) * (size_t)(rows + 1), cudaMemcpyHostToDevice), "upload");
    if (nnz) {
        GK(cudaMemcpy(col, m->col_idx, sizeof(int64_t) * (size_t)nnz, cudaMemcpyHostToDevice), "upload");
        GK(cudaMemcpy(vals, m->values, (size_t)nnz * prec, cudaMemcpyHostToDevice), "upload");
    }
    GK(cudaMemset(head, 0, std::max<int64_t>(nnz, 1)), "memset");
    pt.mark("upload");
    GK(cudaMemset(err, 0, sizeof(unsigned int)), "memset");
    a.row_start = rs;
    a.col = col;
    a.vals = vals;
    a.head = head;
    a.err = err;
    const int grid = sms * 8;
    unsigned int herr = 0;
    // 1. validation + symbols
    Dist ddist, vdist;
    {
        Buffers E;  // keys, freed after the distributions
        uint32_t *dkey;
        uint64_t *vkey;
        GK(E.alloc(&dkey, nnz), "cudaMalloc");
        GK(E.alloc(&vkey, nnz), "cudaMalloc");  // u64 (f64) or u32 (f32) keys
        a.dkey = dkey;
        a.vkey = vkey;
        if (rows) mark_heads<<<grid, 256>>>(a, head);
        if (nnz) {
            if (prec == 8) extract<unsigned long long><<<grid, 256>>>(a);
            else extract<uint32_t><<<grid, 256>>>(a);
        }
        GK(cudaGetLastError(), "launch");
        GK(cudaMemcpy(&herr, err, sizeof(herr), cudaMemcpyDeviceToHost), "download");
        if (herr & kErrRowStart) return fail(DTANS_E_PARAM, "row_start must be nondecreasing");
        if (herr & kErrColRange) return fail(DTANS_E_PARAM, "column index out of range");
        if (herr & kErrColOrder) return fail(DTANS_E_PARAM, "columns must be strictly ascending per row");
        pt.mark("extract");
        // 2. distributions (container.py:112-114)
        int rc = distribution<uint32_t>(E, dkey, nnz, ddist, out);
        if (rc) return rc;
        rc = prec == 8 ? distribution<uint64_t>(E, vkey, nnz, vdist, out)
                       : distribution<uint32_t>(E, reinterpret_cast<uint32_t *>(vkey), nnz, vdist, out);
        if (rc) return rc;
    }
    pt.mark("distributions");
    // 3. quantize + tables on the host
    const int rec = prec == 8 ? 16 : 12;
    out->tables = (uint8_t *)malloc((size_t)kK * rec);
    out->row_symbols = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)std::max<int64_t>(rows, 1));
    out->directory = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(nslices + 1));
    if (!out->tables || !out->row_symbols || !out->directory) {
        dtans_encoded_free(out);
        return fail(DTANS_E_NOMEM, "host allocation failed");
    }
    Domain Dd, Dv;
    {
        const int rc = prepare_tables(ddist, vdist, prec, opts, out->tables, Dd, Dv);
        if (rc) {
            dtans_encoded_free(out);
            return rc;
        }
    }
    pt.mark("quantize+tables");
    for (int64_t i = 0; i < rows; i++) out->row_symbols[i] = (uint32_t)(2 * (m->row_start[i + 1] - m->row_start[i]));
    out->rows = rows;
    out->cols = m->cols;
    out->nnz = nnz;
    out->nslices = nslices;
    out->precision = prec;
    out->rec_size = rec;
    out->directory[0] = 0;
    if (nslices == 0) {
        out->stream = (uint32_t *)malloc(sizeof(uint32_t));
        return DTANS_OK;
    }
    {
        const int rc1 = upload_domain(B, Dd, a.dom[0], out);
        if (rc1) return rc1;
        const int rc2 = upload_domain(B, Dv, a.dom[1], out);
        if (rc2) return rc2;
    }
    const size_t smem = 8 * (size_t)(a.dom[0].nret + a.dom[1].nret);
    GK(cudaFuncSetAttribute(base_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "attr");
    GK(cudaFuncSetAttribute(emit_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "attr");
    // 4. base pass -> flags, slice word counts
    uint64_t *swords, *dir;
    GK(B.alloc(&swords, nslices), "cudaMalloc");
    GK(B.alloc(&dir, nslices + 1), "cudaMalloc");
    a.flags = head;  // the head marks are no longer needed
    a.slice_words = swords;
    const int egrid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * 8, (nslices + 7) / 8));
    base_pass<<<egrid, 256, smem>>>(a);
    GK(cudaGetLastError(), "launch");
    // 5. directory = exclusive scan of the slice word counts
    {
        size_t tb = 0;
        GK(cub::DeviceScan::InclusiveSum(nullptr, tb, swords, dir + 1, nslices), "scan");
        uint8_t *tmp;
        GK(B.alloc(&tmp, tb), "cudaMalloc");
        GK(cub::DeviceScan::InclusiveSum(tmp, tb, swords, dir + 1, nslices), "scan");
        GK(cudaMemset(dir, 0, sizeof(uint64_t)), "memset");
    }
    GK(cudaMemcpy(out->directory, dir, sizeof(uint64_t) * (size_t)(nslices + 1), cudaMemcpyDeviceToHost), "download");
    GK(cudaMemcpy(&herr, err, sizeof(herr), cudaMemcpyDeviceToHost), "download");
    if (herr & kErrCoding) {
        dtans_encoded_free(out);
        return fail(DTANS_E_CODING, "symbol not retained and its table has no escape entry");
    }
    const int64_t nwords = (int64_t)out->directory[nslices];
    pt.mark("base+scan");
    // 6. digit pass + interleave
    uint32_t *stream;
    GK(B.alloc(&stream, nwords), "cudaMalloc");
    a.directory = dir;
    a.stream = stream;
    emit_pass<<<egrid, 256, smem>>>(a);
    GK(cudaGetLastError(), "launch");
    pt.mark("emit");
    out->stream = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)std::max<int64_t>(nwords, 1));
    if (!out->stream) {
        dtans_encoded_free(out);
        return fail(DTANS_E_NOMEM, "host allocation failed");
    }
    GK(cudaMemcpy(out->stream, stream, sizeof(uint32_t) * (size_t)nwords, cudaMemcpyDeviceToHost), "download");
    GK(cudaMemcpy(&herr, err, sizeof(herr), cudaMemcpyDeviceToHost), "download");
    if (herr & kErrCorrupt) {
        dtans_encoded_free(out);
        return fail(DTANS_E_CORRUPT, "GPU encoder: slice word accounting mismatch");
    }
    out->nwords = nwords;
    pt.mark("download");
    return DTANS_OK;
}
