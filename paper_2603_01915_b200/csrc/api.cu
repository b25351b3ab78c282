// C ABI of libdtans.so: device upload, fused SpMV / decode launches.
// Declarations and reference citations: include/dtans.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "checkpoints.h"
#include "common.h"
#include "kernels.cuh"

using namespace dtans;

constexpr int kHostChunks = 8;

struct dtans_dev {
    int device = 0;
    int64_t rows = 0, cols = 0, nnz = 0, nslices = 0, nwords = 0;
    int32_t precision = 8;
    void *d_base = nullptr;     // single allocation for all container arrays
    size_t d_bytes = 0;
    uint32_t *d_tables = nullptr;
    uint32_t *d_row_symbols = nullptr;
    uint64_t *d_directory = nullptr;
    uint32_t *d_stream = nullptr;
    unsigned int *d_err = nullptr;
    // staging buffers for the host-pointer entry point
    void *d_io = nullptr;
    size_t io_bytes = 0;
    dev::KernelArgs base{};     // launch-invariant kernel arguments
    int ctas = 0, threads = 1024, smem = 0;
    int64_t launches = 0;
    int64_t staged_slices = 0;  // slices whose stream fits a ring buffer
    // long-slice checkpoint index
    void *d_long = nullptr;     // tasks + pool + slices + partials
    size_t long_bytes = 0;
    int task_ctas = 0, task_smem = 0, solo_ctas = 0, solo_smem = 0;
    uint32_t *d_row_map = nullptr;  // optional output row map (reordered P*A)
    uint32_t *d_order = nullptr;    // optional longest-first slice order (dynamic scheduling)
    uint64_t long_words = ~0ull;    // slices with a larger aligned window are task-decoded
    // pipelined host path: copy-in, compute, copy-out streams and per-chunk events
    cudaStream_t st_in = nullptr, st_comp = nullptr, st_out = nullptr;
    cudaEvent_t ev_in[kHostChunks] = {}, ev_done[kHostChunks] = {};
};

namespace {

int cuda_fail(cudaError_t e, const char *what)
{
    return fail(DTANS_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define CK(call, what)                                   \
    do {                                                 \
        cudaError_t _e = (call);                         \
        if (_e != cudaSuccess) return cuda_fail(_e, what); \
    } while (0)

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Compact slot tables: entry = digit | (base-1) << 8 | id << 16 with id the
// index of the slot's symbol in the domain dictionary (ascending retained
// symbols) and id = n_retained for escape slots.
struct TableBlock {
    std::vector<uint32_t> words;  // [dtab][vtab][ddict (+pad)][vdict (+pad)]
    int32_t off_ddict = 0, off_vdict = 0;
    uint32_t nd = 0, nv = 0;
};

TableBlock build_table_block(const uint8_t *recs, int precision)
{
    const int rec = precision == 8 ? 16 : 12;
    const uint64_t vsent = precision == 8 ? ~0ull : 0xFFFFFFFFull;
    std::vector<uint64_t> dsym(kK), vsym(kK);
    std::vector<uint8_t> desc(kK), vesc(kK), ddig(kK), dbm1(kK), vdig(kK), vbm1(kK);
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
        dsym[j] = ds;
        vsym[j] = vs;
        desc[j] = ds == (uint32_t)kDeltaSentinel;
        vesc[j] = vs == vsent;
        ddig[j] = r[0];
        dbm1[j] = r[1];
        vdig[j] = r[2];
        vbm1[j] = r[3];
    }
    auto dict = [](const std::vector<uint64_t> &sym, const std::vector<uint8_t> &esc) {
        std::vector<uint64_t> u;
        for (int j = 0; j < kK; j++)
            if (!esc[j]) u.push_back(sym[j]);
        std::sort(u.begin(), u.end());
        u.erase(std::unique(u.begin(), u.end()), u.end());
        return u;
    };
    const std::vector<uint64_t> dd = dict(dsym, desc), vd = dict(vsym, vesc);
    TableBlock tb;
    tb.nd = (uint32_t)dd.size();
    tb.nv = (uint32_t)vd.size();
    const size_t dict_d_words = align_up(dd.size() + 1, 4);
    const size_t vw = precision == 8 ? 2 : 1;
    const size_t dict_v_words = align_up((vd.size() + 1) * vw, 4);
    tb.words.assign(2 * kK + dict_d_words + dict_v_words, 0);
    tb.off_ddict = (int32_t)(2 * kK * 4);
    tb.off_vdict = (int32_t)((2 * kK + dict_d_words) * 4);
    for (int j = 0; j < kK; j++) {
        // id field = byte offset of the symbol in its dictionary; escapes
        // point at the dummy slot after the retained symbols
        const uint32_t did = 4u * (desc[j] ? tb.nd
                                           : (uint32_t)(std::lower_bound(dd.begin(), dd.end(), dsym[j]) - dd.begin()));
        const uint32_t vid = (uint32_t)(4 * vw) *
                             (vesc[j] ? tb.nv
                                      : (uint32_t)(std::lower_bound(vd.begin(), vd.end(), vsym[j]) - vd.begin()));
        tb.words[j] = (uint32_t)ddig[j] | ((uint32_t)dbm1[j] << 8) | (did << 16);
        tb.words[kK + j] = (uint32_t)vdig[j] | ((uint32_t)vbm1[j] << 8) | (vid << 16);
    }
    for (size_t i = 0; i < dd.size(); i++) tb.words[2 * kK + i] = (uint32_t)dd[i];
    uint32_t *vdw = tb.words.data() + 2 * kK + dict_d_words;
    for (size_t i = 0; i < vd.size(); i++) {
        if (vw == 2) {
            vdw[2 * i] = (uint32_t)vd[i];
            vdw[2 * i + 1] = (uint32_t)(vd[i] >> 32);
        } else {
            vdw[i] = (uint32_t)vd[i];
        }
    }
    return tb;
}

// Dispatch on the compile-time CTA size.
template <typename V, class F>
int with_kernel(bool dyn, F &&f)
{
    if (dyn)
        return f(dev::dtans_kernel<V, false, true, true, 1024>, dev::dtans_kernel<V, false, false, true, 1024>,
                 dev::dtans_kernel<V, true, false, true, 1024>);
    return f(dev::dtans_kernel<V, false, true, false, 1024>, dev::dtans_kernel<V, false, false, false, 1024>,
             dev::dtans_kernel<V, true, false, false, 1024>);
}

template <typename V>
int configure(dtans_dev *h, const TableBlock &tb, const uint64_t *directory)
{
    dev::KernelArgs &a = h->base;
    a.tables = h->d_tables;
    a.table_bytes = (int32_t)(tb.words.size() * 4);
    a.off_ddict = tb.off_ddict;
    a.off_vdict = tb.off_vdict;
    a.desc_min = (4u * tb.nd) << 16;
    a.vesc_min = ((uint32_t)(sizeof(V)) * tb.nv) << 16;
    a.pads_ok = tb.nd > 0 && tb.nv > 0;
    a.row_symbols = h->d_row_symbols;
    a.directory = h->d_directory;
    a.stream = h->d_stream;
    a.rows = h->rows;
    a.cols = h->cols;
    a.nslices = h->nslices;
    a.nwords = h->nwords;
    a.err = h->d_err;
    a.work_counter = h->d_err + 8;
    a.slice_lo = 0;
    a.slice_hi = (uint32_t)h->nslices;
    int max_optin = 0, sms = 0;
    if (a.nlong) {
        h->task_smem = (int)align_up((size_t)a.table_bytes, 16);
        h->solo_smem = (int)align_up((size_t)a.table_bytes, 16);
        CK(cudaFuncSetAttribute(dev::dtans_solo_kernel<V, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                h->solo_smem), "cudaFuncSetAttribute");
        CK(cudaFuncSetAttribute(dev::dtans_solo_kernel<V, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                h->solo_smem), "cudaFuncSetAttribute");
        CK(cudaFuncSetAttribute(dev::dtans_task_kernel<V, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                h->task_smem), "cudaFuncSetAttribute");
        CK(cudaFuncSetAttribute(dev::dtans_task_kernel<V, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                h->task_smem), "cudaFuncSetAttribute");
        int per = 0, nsm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, dev::dtans_task_kernel<V, false>, 512, h->task_smem),
           "occupancy");
        CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, h->device), "sm count");
        h->task_ctas = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)nsm * std::max(per, 1),
                                                                    ((int64_t)a.ntasks + 15) / 16));
        int pers = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pers, dev::dtans_solo_kernel<V, false>, 256, h->solo_smem),
           "occupancy");
        h->solo_ctas = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)nsm * std::max(pers, 1),
                                                                    ((int64_t)a.nsolo + 255) / 256));
    }
    CK(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device), "attr");
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device), "sm count");
    size_t off = (size_t)a.table_bytes;
    off = align_up(off, 16);
    a.off_bars = (int32_t)off;
    off += dev::kMaxWarps * dev::kRing * 8;
    off = align_up(off, 16);
    a.off_meta = (int32_t)off;
    off += dev::kMaxWarps * dev::kRing * sizeof(dev::SliceMeta);
    off = align_up(off, 128);
    a.off_bufs = (int32_t)off;
    // ring buffer size: the largest 16-byte-aligned slice window, capped by
    // what fits; bigger slices are decoded straight from global memory.
    uint64_t max_words = 4;
    for (int64_t s = 0; s < h->nslices; s++) {
        const uint64_t lo = directory[s] & ~3ull, hi = (directory[s + 1] + 3) & ~3ull;
        if (hi - lo <= h->long_words) max_words = std::max<uint64_t>(max_words, hi - lo);
    }
    h->threads = 1024;
    const int warps = h->threads / 32;
    const int64_t budget =
        ((int64_t)max_optin - (int64_t)off - dev::kOverrunWords * 4) / (warps * dev::kRing * 4);
    if (budget < 4) return fail(DTANS_E_CUDA, "coding tables leave no shared memory for staging");
    a.bufw = (int32_t)std::min<int64_t>((int64_t)align_up(max_words, 4), budget / 4 * 4);
    h->staged_slices = 0;
    for (int64_t s = 0; s < h->nslices; s++) {
        const uint64_t lo = directory[s] & ~3ull, hi = (directory[s + 1] + 3) & ~3ull;
        if (hi - lo <= (uint64_t)a.bufw) h->staged_slices++;
    }
    h->smem = (int)(off + ((size_t)warps * dev::kRing * a.bufw + dev::kOverrunWords) * 4);
    int per_sm = 0;
    int rc = with_kernel<V>(h->base.dynamic != 0, [&](auto kspmv, auto kspmv0, auto kdec) -> int {
        CK(cudaFuncSetAttribute(kspmv, cudaFuncAttributeMaxDynamicSharedMemorySize, h->smem), "cudaFuncSetAttribute");
        CK(cudaFuncSetAttribute(kspmv0, cudaFuncAttributeMaxDynamicSharedMemorySize, h->smem), "cudaFuncSetAttribute");
        CK(cudaFuncSetAttribute(kdec, cudaFuncAttributeMaxDynamicSharedMemorySize, h->smem), "cudaFuncSetAttribute");
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kspmv, h->threads, h->smem), "occupancy");
        return DTANS_OK;
    });
    if (rc) return rc;
    if (per_sm < 1) return fail(DTANS_E_CUDA, "kernel does not fit on an SM");
    const int64_t ctas_needed = (h->nslices + warps - 1) / warps;
    h->ctas = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * per_sm, ctas_needed));
    return DTANS_OK;
}

template <typename V>
int launch(dtans_dev *h, const V *x, const V *y, V *out, const int64_t *row_start, int64_t *cols,
           void *vals, bool decode_only, cudaStream_t st, int64_t s_lo = -1, int64_t s_hi = -1)
{
    if (h->nslices == 0) return DTANS_OK;
    dev::KernelArgs a = h->base;
    int ctas = h->ctas;
    if (s_lo >= 0) {  // slice range (pipelined host path; static order, no long slices)
        a.slice_lo = (uint32_t)s_lo;
        a.slice_hi = (uint32_t)s_hi;
        ctas = (int)std::max<int64_t>(1, std::min<int64_t>(h->ctas, (s_hi - s_lo + 31) / 32));
    }
    if (a.dynamic) CK(cudaMemsetAsync(a.work_counter, 0, sizeof(uint32_t), st), "reset work counter");
    a.x = x;
    a.y = y;
    a.out = out;
    a.row_start = row_start;
    a.dec_cols = cols;
    a.dec_vals = vals;
    with_kernel<V>(a.dynamic != 0, [&](auto kspmv, auto kspmv0, auto kdec) -> int {
        if (decode_only)
            kdec<<<ctas, h->threads, h->smem, st>>>(a);
        else if (y != nullptr)
            kspmv<<<ctas, h->threads, h->smem, st>>>(a);
        else
            kspmv0<<<ctas, h->threads, h->smem, st>>>(a);
        return 0;
    });
    h->launches++;
    if (a.nlong) {
        if (decode_only) {
            if (a.ntasks) dev::dtans_task_kernel<V, true><<<h->task_ctas, 512, h->task_smem, st>>>(a);
            if (a.nsolo) dev::dtans_solo_kernel<V, true><<<h->solo_ctas, 256, h->solo_smem, st>>>(a);
            h->launches += (a.ntasks ? 1 : 0) + (a.nsolo ? 1 : 0);
        } else {
            if (a.ntasks) dev::dtans_task_kernel<V, false><<<h->task_ctas, 512, h->task_smem, st>>>(a);
            if (a.nsolo) dev::dtans_solo_kernel<V, false><<<h->solo_ctas, 256, h->solo_smem, st>>>(a);
            const unsigned nb = a.nlong_small_blocks + (a.nlong - a.nlong_small);
            if (y != nullptr)
                dev::dtans_finalize_kernel<V, true><<<nb, 256, 0, st>>>(a);
            else
                dev::dtans_finalize_kernel<V, false><<<nb, 256, 0, st>>>(a);
            h->launches += (a.ntasks ? 1 : 0) + (a.nsolo ? 1 : 0) + 1;
        }
    }
    CK(cudaGetLastError(), "kernel launch");
    return DTANS_OK;
}

}  // namespace

extern "C" int dtans_upload(const dtans_container_view *c, int device, dtans_dev **out)
{
    if (!c || !out) return fail(DTANS_E_PARAM, "null argument");
    *out = nullptr;
    if (c->precision != 4 && c->precision != 8) return fail(DTANS_E_PARAM, "precision must be 4 or 8");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(DTANS_E_NODEVICE, "no CUDA device visible: the dtANS SpMV has no CPU path");
    }
    if (device < 0 || device >= ndev) return fail(DTANS_E_PARAM, "bad device ordinal %d", device);
    CK(cudaSetDevice(device), "cudaSetDevice");
    if (c->rows >= ((int64_t)1 << 32)) return fail(DTANS_E_PARAM, "the device path needs rows < 2^32");
    const int64_t nsl = (c->rows + kSlice - 1) / kSlice;
    if (c->nslices != nsl) return fail(DTANS_E_PARAM, "nslices does not match rows");
    if ((int64_t)c->directory[nsl] != c->nwords)
        return fail(DTANS_E_CORRUPT, "directory does not span the stream");

    dtans_dev *h = new dtans_dev();
    h->device = device;
    h->rows = c->rows;
    h->cols = c->cols;
    h->nnz = c->nnz;
    h->nslices = nsl;
    h->nwords = c->nwords;
    h->precision = c->precision;
    const TableBlock tb = build_table_block(c->tables, c->precision);
    LongIndex li;
    {
        const char *e1 = getenv("DTANS_LONG_SEG"), *e2 = getenv("DTANS_CHUNK");
        const int long_seg = e1 ? atoi(e1) : 64, chunk = e2 ? atoi(e2) : 32;
        // slices whose stream window cannot be staged in a ring buffer go to
        // the task kernels as well (their words would be read uncached)
        int max_optin = 0;
        if (cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) != cudaSuccess)
            max_optin = 227 * 1024;
        const int64_t fixed = (int64_t)tb.words.size() * 4 + dev::kMaxWarps * dev::kRing * (8 + sizeof(dev::SliceMeta)) +
                              256 + dev::kOverrunWords * 4;
        const uint64_t max_words = (uint64_t)std::max<int64_t>(4, (max_optin - fixed) / (dev::kMaxWarps * dev::kRing * 4) / 4 * 4);
        const int rc0 = build_long_index(c, long_seg, max_words, std::max(1, chunk), li);
        if (rc0) {
            delete h;
            return rc0;
        }
        h->base.long_seg = li.slices.empty() ? 0xFFFFFFFFu : (uint32_t)long_seg;
        h->long_words = max_words;
        h->base.long_words = li.slices.empty() ? 0xFFFFFFFFu : (uint32_t)std::min<uint64_t>(max_words, 0xFFFFFFFEull);
        h->base.ntasks = (uint32_t)li.tasks.size();
        h->base.nsolo = (uint32_t)li.solo.size();
        h->base.nlong = (uint32_t)li.slices.size();
        uint32_t small = 0;
        while (small < li.slices.size() && li.slices[small].nparts <= 32) small++;
        h->base.nlong_small = small;
        h->base.nlong_small_blocks = (small + 7) / 8;
        h->base.single_direct = 1;
    }

    // one allocation: [tables][row_symbols][directory][stream + pad][err]
    size_t off = 0;
    const size_t o_tb = off; off = align_up(off + tb.words.size() * 4, 256);
    const size_t o_rs = off; off = align_up(off + sizeof(uint32_t) * (size_t)std::max<int64_t>(c->rows, 1), 256);
    const size_t o_di = off; off = align_up(off + sizeof(uint64_t) * (size_t)(nsl + 1), 256);
    const size_t o_st = off; off = align_up(off + sizeof(uint32_t) * ((size_t)c->nwords + dev::kStreamPadWords), 256);
    const size_t o_er = off; off = align_up(off + 64, 256);
    cudaError_t e = cudaMalloc(&h->d_base, off);
    if (e != cudaSuccess) {
        delete h;
        return fail(DTANS_E_NOMEM, "cudaMalloc(%zu): %s", off, cudaGetErrorString(e));
    }
    h->d_bytes = off;
    char *b = (char *)h->d_base;
    h->d_tables = (uint32_t *)(b + o_tb);
    h->d_row_symbols = (uint32_t *)(b + o_rs);
    h->d_directory = (uint64_t *)(b + o_di);
    h->d_stream = (uint32_t *)(b + o_st);
    h->d_err = (unsigned int *)(b + o_er);
    int rc = DTANS_OK;
    auto cp = [&](void *dst, const void *src, size_t n) {
        if (rc == DTANS_OK && n) {
            cudaError_t ce = cudaMemcpy(dst, src, n, cudaMemcpyHostToDevice);
            if (ce != cudaSuccess) rc = cuda_fail(ce, "upload");
        }
    };
    cp(h->d_tables, tb.words.data(), tb.words.size() * 4);
    cp(h->d_row_symbols, c->row_symbols, sizeof(uint32_t) * (size_t)c->rows);
    cp(h->d_directory, c->directory, sizeof(uint64_t) * (size_t)(nsl + 1));
    cp(h->d_stream, c->stream, sizeof(uint32_t) * (size_t)c->nwords);
    if (rc == DTANS_OK) {
        cudaError_t ce = cudaMemset(h->d_stream + c->nwords, 0, sizeof(uint32_t) * dev::kStreamPadWords);
        if (ce == cudaSuccess) ce = cudaMemset(h->d_err, 0, 64);
        if (ce != cudaSuccess) rc = cuda_fail(ce, "memset");
    }
    if (rc == DTANS_OK && !li.slices.empty()) {
        const size_t tb_b = align_up(li.tasks.size() * sizeof(LongTask), 256) +
                            align_up(li.solo.size() * sizeof(SoloTask), 256);
        const size_t pl_b = align_up(li.pool.size() * 4, 256);
        const size_t ls_b = align_up(li.slices.size() * sizeof(LongSlice), 256);
        const size_t pa_b = align_up((size_t)li.nparts * 32 * c->precision, 256);
        h->long_bytes = tb_b + pl_b + ls_b + pa_b;
        cudaError_t ce = cudaMalloc(&h->d_long, h->long_bytes);
        if (ce != cudaSuccess) {
            rc = fail(DTANS_E_NOMEM, "cudaMalloc(long index): %s", cudaGetErrorString(ce));
        } else {
            char *lb = (char *)h->d_long;
            h->base.tasks = (const LongTask *)lb;
            h->base.solo = (const SoloTask *)(lb + align_up(li.tasks.size() * sizeof(LongTask), 256));
            h->base.ck_pool = (const uint32_t *)(lb + tb_b);
            h->base.longs = (const LongSlice *)(lb + tb_b + pl_b);
            h->base.partials = lb + tb_b + pl_b + ls_b;
            cp(lb, li.tasks.data(), li.tasks.size() * sizeof(LongTask));
            cp((void *)h->base.solo, li.solo.data(), li.solo.size() * sizeof(SoloTask));
            if (rc == DTANS_OK) {
                // partial slots of solo tasks are written for one lane only
                cudaError_t me = cudaMemset(h->base.partials, 0, pa_b);
                if (me != cudaSuccess) rc = cuda_fail(me, "memset partials");
            }
            cp(lb + tb_b, li.pool.data(), li.pool.size() * 4);
            cp(lb + tb_b + pl_b, li.slices.data(), li.slices.size() * sizeof(LongSlice));
        }
    }
    if (rc == DTANS_OK && nsl > 0) {
        // skewed slice costs -> dynamic longest-first scheduling
        std::vector<uint32_t> cost((size_t)nsl);
        double mean = 0;
        uint32_t mx = 0;
        for (int64_t s = 0; s < nsl; s++) {
            uint32_t m = 0;
            for (int64_t i = s * kSlice; i < std::min<int64_t>((s + 1) * kSlice, c->rows); i++)
                m = std::max(m, c->row_symbols[i]);
            cost[s] = (m + 7) / 8;
            const uint64_t words = ((c->directory[s + 1] + 3) & ~3ull) - (c->directory[s] & ~3ull);
            if (cost[s] > h->base.long_seg || words > h->long_words) cost[s] = 0;  // task-decoded
            mean += cost[s];
            mx = std::max(mx, cost[s]);
        }
        mean /= (double)nsl;
        const char *ed = getenv("DTANS_DYNAMIC");
        const bool dyn = ed ? atoi(ed) != 0 : (mx > 4.0 * std::max(mean, 1.0));
        h->base.dynamic = dyn ? 1 : 0;
        bool sorted = true;
        for (int64_t s = 1; s < nsl && sorted; s++) sorted = cost[s] <= cost[s - 1];
        if (dyn && !sorted) {
            std::vector<uint32_t> order((size_t)nsl);
            for (int64_t s = 0; s < nsl; s++) order[s] = (uint32_t)s;
            std::stable_sort(order.begin(), order.end(), [&](uint32_t p, uint32_t q) { return cost[p] > cost[q]; });
            cudaError_t ce = cudaMalloc(&h->d_order, sizeof(uint32_t) * order.size());
            if (ce != cudaSuccess) rc = cuda_fail(ce, "cudaMalloc slice order");
            else {
                cp(h->d_order, order.data(), sizeof(uint32_t) * order.size());
                h->base.slice_order = h->d_order;
            }
        }
    }
    if (rc == DTANS_OK)
        rc = c->precision == 8 ? configure<double>(h, tb, c->directory) : configure<float>(h, tb, c->directory);
    if (rc != DTANS_OK) {
        cudaFree(h->d_base);
        if (h->d_long) cudaFree(h->d_long);
        if (h->d_order) cudaFree(h->d_order);
        delete h;
        return rc;
    }
    *out = h;
    return DTANS_OK;
}

extern "C" void dtans_free(dtans_dev *h)
{
    if (!h) return;
    cudaSetDevice(h->device);
    if (h->d_base) cudaFree(h->d_base);
    if (h->d_long) cudaFree(h->d_long);
    if (h->d_row_map) cudaFree(h->d_row_map);
    if (h->d_order) cudaFree(h->d_order);
    if (h->d_io) cudaFree(h->d_io);
    for (int k = 0; k < kHostChunks; k++) {
        if (h->ev_in[k]) cudaEventDestroy(h->ev_in[k]);
        if (h->ev_done[k]) cudaEventDestroy(h->ev_done[k]);
    }
    if (h->st_in) cudaStreamDestroy(h->st_in);
    if (h->st_comp) cudaStreamDestroy(h->st_comp);
    if (h->st_out) cudaStreamDestroy(h->st_out);
    delete h;
}

extern "C" int dtans_info(const dtans_dev *h, int64_t *device_bytes, int32_t *ctas,
                          int32_t *warps_per_cta, int32_t *smem_bytes)
{
    if (!h) return fail(DTANS_E_PARAM, "null handle");
    if (device_bytes) *device_bytes = (int64_t)(h->d_bytes + h->long_bytes);
    if (ctas) *ctas = h->ctas;
    if (warps_per_cta) *warps_per_cta = h->threads / 32;
    if (smem_bytes) *smem_bytes = h->smem;
    return DTANS_OK;
}

extern "C" int dtans_set_row_map(dtans_dev *h, const uint32_t *host_map)
{
    if (!h) return fail(DTANS_E_PARAM, "null handle");
    CK(cudaSetDevice(h->device), "cudaSetDevice");
    if (!host_map) {
        if (h->d_row_map) cudaFree(h->d_row_map);
        h->d_row_map = nullptr;
        h->base.row_map = nullptr;
        return DTANS_OK;
    }
    std::vector<uint8_t> seen((size_t)h->rows, 0);
    for (int64_t i = 0; i < h->rows; i++) {
        if (host_map[i] >= (uint64_t)h->rows || seen[host_map[i]])
            return fail(DTANS_E_PARAM, "row map must be a permutation of [0, rows)");
        seen[host_map[i]] = 1;
    }
    if (!h->d_row_map) CK(cudaMalloc(&h->d_row_map, sizeof(uint32_t) * (size_t)std::max<int64_t>(h->rows, 1)), "cudaMalloc row map");
    CK(cudaMemcpy(h->d_row_map, host_map, sizeof(uint32_t) * (size_t)h->rows, cudaMemcpyHostToDevice), "upload row map");
    h->base.row_map = h->d_row_map;
    return DTANS_OK;
}

extern "C" int64_t dtans_launch_count(const dtans_dev *h) { return h ? h->launches : 0; }

extern "C" int dtans_spmv_f64(dtans_dev *h, const double *x, const double *y, double *out,
                              void *stream)
{
    if (!h) return fail(DTANS_E_PARAM, "null handle");
    if (h->precision != 8) return fail(DTANS_E_PARAM, "container precision is f32");
    CK(cudaSetDevice(h->device), "cudaSetDevice");
    return launch<double>(h, x, y, out, nullptr, nullptr, nullptr, false, (cudaStream_t)stream);
}

extern "C" int dtans_spmv_f32(dtans_dev *h, const float *x, const float *y, float *out,
                              void *stream)
{
    if (!h) return fail(DTANS_E_PARAM, "null handle");
    if (h->precision != 4) return fail(DTANS_E_PARAM, "container precision is f64");
    CK(cudaSetDevice(h->device), "cudaSetDevice");
    return launch<float>(h, x, y, out, nullptr, nullptr, nullptr, false, (cudaStream_t)stream);
}

extern "C" int dtans_check(dtans_dev *h, void *stream)
{
    if (!h) return fail(DTANS_E_PARAM, "null handle");
    CK(cudaSetDevice(h->device), "cudaSetDevice");
    CK(cudaStreamSynchronize((cudaStream_t)stream), "synchronize");
    unsigned int err = 0;
    CK(cudaMemcpy(&err, h->d_err, sizeof(err), cudaMemcpyDeviceToHost), "read error word");
    if (err) {
        CK(cudaMemset(h->d_err, 0, sizeof(err)), "clear error word");
        if (err & 1u) return fail(DTANS_E_CORRUPT, "slice consumed an unexpected number of words");
        return fail(DTANS_E_CORRUPT, "decoded column index out of range");
    }
    return DTANS_OK;
}

extern "C" int dtans_spmv_host(dtans_dev *h, const void *x, const void *y, void *out)
{
    if (!h) return fail(DTANS_E_PARAM, "null handle");
    CK(cudaSetDevice(h->device), "cudaSetDevice");
    const size_t es = (size_t)h->precision;
    const size_t xb = align_up(es * (size_t)std::max<int64_t>(h->cols, 1), 256);
    const size_t yb = align_up(es * (size_t)std::max<int64_t>(h->rows, 1), 256);
    const size_t need = xb + 2 * yb;
    if (h->io_bytes < need) {
        if (h->d_io) cudaFree(h->d_io);
        h->d_io = nullptr;
        h->io_bytes = 0;
        CK(cudaMalloc(&h->d_io, need), "cudaMalloc io");
        h->io_bytes = need;
    }
    char *dx = (char *)h->d_io, *dy = dx + xb, *dout = dy + yb;
    // Pipelined: x in, then per slice-range chunk y in (copy-in stream), the
    // kernel on that range (compute stream) and y' out (copy-out stream), so
    // the D2H of a chunk overlaps the H2D and decode of the next.  Containers
    // with long slices or dynamic scheduling use one launch.
    const bool chunked = h->base.nlong == 0 && !h->base.dynamic && h->nslices >= 64 * kHostChunks;
    if (!h->st_in) {
        CK(cudaStreamCreateWithFlags(&h->st_in, cudaStreamNonBlocking), "stream");
        CK(cudaStreamCreateWithFlags(&h->st_comp, cudaStreamNonBlocking), "stream");
        CK(cudaStreamCreateWithFlags(&h->st_out, cudaStreamNonBlocking), "stream");
        for (int k = 0; k < kHostChunks; k++) {
            CK(cudaEventCreateWithFlags(&h->ev_in[k], cudaEventDisableTiming), "event");
            CK(cudaEventCreateWithFlags(&h->ev_done[k], cudaEventDisableTiming), "event");
        }
    }
    const int nch = chunked ? kHostChunks : 1;
    CK(cudaMemcpyAsync(dx, x, es * (size_t)h->cols, cudaMemcpyHostToDevice, h->st_in), "H2D x");
    for (int k = 0; k < nch; k++) {
        const int64_t s0 = h->nslices * k / nch, s1 = h->nslices * (k + 1) / nch;
        const int64_t r0 = s0 * kSlice, r1 = std::min<int64_t>(s1 * kSlice, h->rows);
        if (y && r1 > r0)
            CK(cudaMemcpyAsync(dy + es * r0, (const char *)y + es * r0, es * (size_t)(r1 - r0),
                               cudaMemcpyHostToDevice, h->st_in), "H2D y");
        CK(cudaEventRecord(h->ev_in[k], h->st_in), "event");
        CK(cudaStreamWaitEvent(h->st_comp, h->ev_in[k], 0), "wait");
        int rc;
        const int64_t lo = chunked ? s0 : -1, hi = chunked ? s1 : -1;
        if (h->precision == 8)
            rc = launch<double>(h, (const double *)dx, y ? (const double *)dy : nullptr, (double *)dout,
                                nullptr, nullptr, nullptr, false, h->st_comp, lo, hi);
        else
            rc = launch<float>(h, (const float *)dx, y ? (const float *)dy : nullptr, (float *)dout,
                               nullptr, nullptr, nullptr, false, h->st_comp, lo, hi);
        if (rc) return rc;
        CK(cudaEventRecord(h->ev_done[k], h->st_comp), "event");
        CK(cudaStreamWaitEvent(h->st_out, h->ev_done[k], 0), "wait");
        const int64_t q0 = chunked ? r0 : 0, q1 = chunked ? r1 : h->rows;
        if (q1 > q0)
            CK(cudaMemcpyAsync((char *)out + es * q0, dout + es * q0, es * (size_t)(q1 - q0),
                               cudaMemcpyDeviceToHost, h->st_out), "D2H out");
    }
    CK(cudaStreamSynchronize(h->st_out), "synchronize");
    return dtans_check(h, h->st_comp);
}

extern "C" int dtans_decode(dtans_dev *h, const int64_t *row_start, int64_t *cols, void *valbits,
                            void *stream)
{
    if (!h) return fail(DTANS_E_PARAM, "null handle");
    CK(cudaSetDevice(h->device), "cudaSetDevice");
    if (h->precision == 8)
        return launch<double>(h, nullptr, nullptr, nullptr, row_start, cols, valbits, true,
                              (cudaStream_t)stream);
    return launch<float>(h, nullptr, nullptr, nullptr, row_start, cols, valbits, true,
                         (cudaStream_t)stream);
}
