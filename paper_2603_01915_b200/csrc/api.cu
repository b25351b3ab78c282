// C ABI of libdtans.so: device upload, fused SpMV / decode launches.
// Declarations and reference citations: include/dtans.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <vector>

#include "checkpoints.h"
#include "common.h"
#include "kernels.cuh"

using namespace dtans;

constexpr int kHostChunks = 32;  // max pipeline stages of the host-buffer path
constexpr size_t kRawStreamPad = dev::kStreamPadWords;

struct dtans_dev {
    int device = 0;
    int64_t rows = 0, cols = 0, nnz = 0, nslices = 0, nwords = 0;
    int32_t precision = 8;
    void *d_base = nullptr;     // single allocation for all container arrays
    size_t d_bytes = 0;
    uint32_t *d_tables = nullptr;
    uint32_t *d_blob = nullptr;     // chunk blobs (kernels.cuh ChunkRec)
    uint64_t blob_words = 0;
    uint32_t *d_row_symbols = nullptr;
    uint64_t *d_directory = nullptr;
    uint32_t *d_stream = nullptr;
    unsigned int *d_err = nullptr;
    // staging buffers for the host-pointer entry point
    void *d_io = nullptr;
    size_t io_bytes = 0;
    dev::KernelArgs base{};     // launch-invariant kernel arguments
    int ctas = 0, threads = 1024, smem = 0;
    int warps = dev::kMaxWarps;  // warps per CTA of the main kernel
    int64_t launches = 0;
    int64_t staged_slices = 0;  // slices whose stream fits a ring buffer
    bool pend = false;          // main kernel instantiation with pending products (kernels.cuh kPend)
    int pdl = 2;                // programmatic dependent launch: 1 main -> task -> solo -> finalize,
                                // 2 task -> solo -> finalize only, 0 off
    bool host_walk = false;     // long-slice index walked on the host (DTANS_GPU_WALK=0)
    void *stager = nullptr;     // HostStager: pinned staging of pageable host buffers (dtans_spmv_host)
    unsigned int *h_err = nullptr;  // pinned copy of the error word (host-buffer path)
    std::vector<uint32_t> split_slices;  // slices whose rows sum several task partials
    size_t upload_staged_bytes = 0;  // bytes streamed through the pinned upload buffers
    int64_t upload_batches = 0;
    // long-slice checkpoint index
    void *d_long = nullptr;     // tasks + pool + slices + partials
    size_t long_bytes = 0;
    int task_ctas = 0, task_smem = 0, solo_ctas = 0, solo_smem = 0;
    uint32_t final_big = 0;     // long slices with > 32 partials (a finalize CTA each)
    uint32_t *d_empty = nullptr;  // all-empty slices (dtans_empty_kernel)
    bool pdl_main = true;       // DTANS_PDL_MAIN: main kernel launched with PDL (overlaps the previous one's tail)
    bool solo_first = true;     // DTANS_SOLO_FIRST: solo kernel first, tasks beside it by ticket
    uint32_t *d_row_map = nullptr;  // optional output row map (reordered P*A)
    uint32_t *d_col_map = nullptr;  // optional column map (symmetric P*A*P^T): x'[j] = x[map[j]]
    void *d_xperm = nullptr;        // x' scratch (cols values)
    std::vector<dev::ChunkRec> chunks;  // work list of the main kernel (host copy)
    dev::ChunkRec *d_chunks = nullptr;
    bool dinline = false;           // delta symbols inline in the slot table
    int sms = 0;
    // pipelined host path: copy-in, compute, copy-out streams and per-chunk events
    cudaStream_t st_in = nullptr, st_comp = nullptr, st_out = nullptr;
    cudaEvent_t ev_in[kHostChunks] = {}, ev_done[kHostChunks] = {};
};

namespace dtans {
void dev_shape(const dtans_dev *h, int64_t *rows, int64_t *cols, int32_t *precision)
{
    *rows = h->rows;
    *cols = h->cols;
    *precision = h->precision;
}
}  // namespace dtans

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

// Shared-memory table image: [dtab u32 4096][vtab u32 4096][ddict][vdict].
// Entry = digit | (base-1) << 8 | F << 16.  Value domain: F = byte offset of
// the symbol in the replicated value dictionary (id * rep_v * width; escapes
// point at the dummy element nv).  Delta domain: inline (every retained
// delta < 0xFFFF): F = the delta, 0xFFFF for escapes; otherwise F = byte
// offset in the replicated delta dictionary.  Dictionaries hold the retained
// symbols ascending; element e of copy c lives at (e * rep + c) * width.
struct TableBlock {
    std::vector<uint32_t> tabs;                // [dtab 4096][vtab 4096]
    std::vector<uint8_t> ddict, vdict;         // replicated dictionaries (16-byte padded)
    int32_t off_ddict = 0, off_vdict = 0;
    int32_t rep_d = 1, rep_v = 1;
    uint32_t nd = 0, nv = 0;
    uint32_t desc_min = 0, vesc_min = 0;
    bool dinline = false;
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
    tb.dinline = dd.empty() || dd.back() < 0xFFFFull;
    const char *ei = getenv("DTANS_DINLINE");
    if (ei && atoi(ei) == 0) tb.dinline = false;
    const uint32_t vw = (uint32_t)precision;  // value width in bytes
    // replication: conflict-free dictionary reads need 32 lanes x width
    // bytes = all 32 banks per wavefront; keep F < 2^16 and each dictionary
    // within a shared-memory budget
    auto pick_rep = [](uint32_t n_el, uint32_t w, uint32_t rmax, uint32_t budget) {
        uint32_t r = rmax;
        while (r > 1 && ((uint64_t)(n_el + 1) * r * w > 65536u || (uint64_t)(n_el + 1) * r * w > budget)) r >>= 1;
        return r;
    };
    const char *er = getenv("DTANS_REP");
    const uint32_t rcap = er ? (uint32_t)std::max(1, atoi(er)) : 32u;
    tb.rep_v = (int32_t)pick_rep(tb.nv, vw, std::min<uint32_t>(rcap, 128u / vw), 36u * 1024u);
    const char *edk = getenv("DTANS_DDICT_KB");  // shared-memory budget of the replicated delta dictionary
    const uint32_t dbudget = (edk ? (uint32_t)std::max(1, atoi(edk)) : 8u) * 1024u;
    tb.rep_d = tb.dinline ? 1 : (int32_t)pick_rep(tb.nd, 4, std::min<uint32_t>(rcap, 32u), dbudget);
    const size_t dict_d_bytes = tb.dinline ? 0 : align_up((size_t)(tb.nd + 1) * tb.rep_d * 4, 16);
    const size_t dict_v_bytes = align_up((size_t)(tb.nv + 1) * tb.rep_v * vw, 16);
    tb.tabs.assign(2 * kK, 0);
    tb.ddict.assign(dict_d_bytes, 0);
    tb.vdict.assign(dict_v_bytes, 0);
    for (int j = 0; j < kK; j++) {
        uint32_t fd;
        if (tb.dinline)
            fd = desc[j] ? 0xFFFFu : (uint32_t)dsym[j];
        else
            fd = 4u * (uint32_t)tb.rep_d *
                 (desc[j] ? tb.nd : (uint32_t)(std::lower_bound(dd.begin(), dd.end(), dsym[j]) - dd.begin()));
        const uint32_t fv = vw * (uint32_t)tb.rep_v *
                            (vesc[j] ? tb.nv : (uint32_t)(std::lower_bound(vd.begin(), vd.end(), vsym[j]) - vd.begin()));
        tb.tabs[j] = (uint32_t)ddig[j] | ((uint32_t)dbm1[j] << 8) | (fd << 16);
        tb.tabs[kK + j] = (uint32_t)vdig[j] | ((uint32_t)vbm1[j] << 8) | (fv << 16);
    }
    tb.desc_min = tb.dinline ? dev::kDeltaInlineEsc : (4u * (uint32_t)tb.rep_d * tb.nd) << 16;
    tb.vesc_min = (vw * (uint32_t)tb.rep_v * tb.nv) << 16;
    if (!tb.dinline)
        for (size_t e = 0; e < dd.size(); e++)
            for (int c = 0; c < tb.rep_d; c++) {
                const uint32_t v = (uint32_t)dd[e];
                memcpy(tb.ddict.data() + (e * tb.rep_d + c) * 4, &v, 4);
            }
    for (size_t e = 0; e < vd.size(); e++)
        for (int c = 0; c < tb.rep_v; c++) {
            if (vw == 8)
                memcpy(tb.vdict.data() + (e * tb.rep_v + c) * 8, &vd[e], 8);
            else {
                const uint32_t v = (uint32_t)vd[e];
                memcpy(tb.vdict.data() + (e * tb.rep_v + c) * 4, &v, 4);
            }
        }
    return tb;
}

// Shared-memory plan (dynamic smem offsets; the dynamic window starts at
// shared address 0x400 mod 16 KB on sm_90+/sm_100, which the kernels check):
//   [bars][metas][warp ctl][low dictionaries]   below kTabOff
//   [delta slot table][value slot table]         at kTabOff (16 KB aligned address)
//   [other dictionaries][staging rings][overrun slack]
// The global table image mirrors [off_img, end of dictionaries).
constexpr int32_t kTabOff = 0x3C00;
struct SmemPlan {
    int32_t off_bars = 0, off_meta = 0, off_ctl = 0, off_bufs = 0, bufb = 0, nring = 3, total = 0;
    int32_t off_img = 0, off_tab = kTabOff, off_ddict = 0, off_vdict = 0;
    std::vector<uint32_t> image;
};

SmemPlan plan_smem(const TableBlock &tb, int max_optin, int nring, int warps)
{
    SmemPlan p;
    p.off_bars = 0;
    p.off_meta = dev::kMaxWarps * dev::kMaxRing * 8;
    p.off_ctl = 2 * dev::kMaxWarps * dev::kMaxRing * 8;
    size_t low = (size_t)p.off_ctl + dev::kMaxWarps * sizeof(dev::WarpCtl);
    const size_t low0 = low;
    size_t high = (size_t)kTabOff + dev::kTabBytes;
    auto place = [&](size_t bytes) -> int32_t {
        if (bytes == 0) return (int32_t)low;
        if (low + bytes <= (size_t)kTabOff) {
            low += bytes;
            return (int32_t)(low - bytes);
        }
        high += bytes;
        return (int32_t)(high - bytes);
    };
    // the larger dictionary first gets the free space below the tables
    if (tb.vdict.size() >= tb.ddict.size()) {
        p.off_vdict = place(tb.vdict.size());
        p.off_ddict = place(tb.ddict.size());
    } else {
        p.off_ddict = place(tb.ddict.size());
        p.off_vdict = place(tb.vdict.size());
    }
    p.off_img = low > low0 ? (int32_t)low0 : kTabOff;
    p.image.assign((high - (size_t)p.off_img) / 4, 0);
    uint8_t *img = reinterpret_cast<uint8_t *>(p.image.data());
    memcpy(img + (kTabOff - p.off_img), tb.tabs.data(), dev::kTabBytes);
    if (!tb.ddict.empty()) memcpy(img + (p.off_ddict - p.off_img), tb.ddict.data(), tb.ddict.size());
    memcpy(img + (p.off_vdict - p.off_img), tb.vdict.data(), tb.vdict.size());
    const size_t off = align_up(high, 128);
    p.off_bufs = (int32_t)off;
    const int64_t avail = (int64_t)max_optin - (int64_t)off - dev::kOverrunWords * 4;
    p.nring = nring;
    p.bufb = (int32_t)std::max<int64_t>(0, avail / (warps * nring) / 16 * 16);
    p.total = (int32_t)(off + (size_t)warps * nring * p.bufb + dev::kOverrunWords * 4);
    return p;
}

// words of the blob of a chunk of slices [s0, s0+k) (kernels.cuh ChunkRec)
uint64_t chunk_words(const uint64_t *dir, int64_t s0, int64_t k)
{
    return dev::chunk_hdr_words((uint32_t)k) + (uint64_t)k * 32 + ((dir[s0 + k] - dir[s0] + 3) & ~3ull);
}
uint64_t chunk_bytes(const uint64_t *dir, int64_t s0, int64_t k) { return 4 * chunk_words(dir, s0, k); }

// Dispatch on the delta-dictionary mode and on the pending-products
// instantiation: (spmv, y-less spmv, decode, scaled y-less spmv).
template <typename V, bool kT, class F>
int with_kernel_t(bool dinline, F &&f)
{
    if (dinline)
        return f(dev::dtans_kernel<V, false, true, true, false, kT>, dev::dtans_kernel<V, false, false, true, false, kT>,
                 dev::dtans_kernel<V, true, false, true, false, kT>, dev::dtans_kernel<V, false, false, true, true, kT>);
    return f(dev::dtans_kernel<V, false, true, false, false, kT>, dev::dtans_kernel<V, false, false, false, false, kT>,
             dev::dtans_kernel<V, true, false, false, false, kT>, dev::dtans_kernel<V, false, false, false, true, kT>);
}
template <typename V, class F>
int with_kernel(bool dinline, bool pend, F &&f)
{
    return pend ? with_kernel_t<V, true>(dinline, f) : with_kernel_t<V, false>(dinline, f);
}

template <typename V, class F>
int with_long_kernels(bool dinline, F &&f)
{
    if (dinline)
        return f(dev::dtans_task_kernel<V, false, true>, dev::dtans_task_kernel<V, true, true>,
                 dev::dtans_solo_kernel<V, false, true>, dev::dtans_solo_kernel<V, true, true>);
    return f(dev::dtans_task_kernel<V, false, false>, dev::dtans_task_kernel<V, true, false>,
             dev::dtans_solo_kernel<V, false, false>, dev::dtans_solo_kernel<V, true, false>);
}

// The launch-invariant kernel arguments of the handle.
void fill_args(dtans_dev *h, const TableBlock &tb, const SmemPlan &sp)
{
    dev::KernelArgs &a = h->base;
    a.tables = h->d_tables;
    a.table_bytes = (int32_t)(sp.image.size() * 4);
    a.off_img = sp.off_img;
    a.off_tab = sp.off_tab;
    a.off_ddict = sp.off_ddict;
    a.off_vdict = sp.off_vdict;
    a.rep_d = tb.rep_d;
    a.rep_v = tb.rep_v;
    a.desc_min = tb.desc_min;
    a.vesc_min = tb.vesc_min;
    a.pads_ok = tb.nd > 0 && tb.nv > 0;
    a.blob = h->d_blob;
    a.row_symbols = h->d_row_symbols;
    a.directory = h->d_directory;
    a.stream = h->d_stream;
    a.rows = h->rows;
    a.cols = h->cols;
    a.nslices = h->nslices;
    a.nwords = h->nwords;
    a.err = h->d_err;
    a.work_counter = h->d_err + 8;
    a.off_bars = sp.off_bars;
    a.off_meta = sp.off_meta;
    a.off_ctl = sp.off_ctl;
    a.off_bufs = sp.off_bufs;
    a.bufb = sp.bufb;
    a.nring = sp.nring;
    a.chunks = h->d_chunks;
    a.chunk_lo = 0;
    a.chunk_hi = (uint32_t)h->chunks.size();
    h->dinline = tb.dinline;
}

template <typename V>
int configure(dtans_dev *h, const TableBlock &tb, const SmemPlan &sp)
{
    dev::KernelArgs &a = h->base;
    fill_args(h, tb, sp);
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device), "sm count");
    h->sms = sms;
    if (a.nlong) {
        h->task_smem = (int)align_up((size_t)(a.off_img + a.table_bytes), 16);
        h->solo_smem = (int)align_up((size_t)(a.off_img + a.table_bytes), 16);
        int per = 0, pers = 0;
        int rc = with_long_kernels<V>(tb.dinline, [&](auto kt, auto ktd, auto ks, auto ksd) -> int {
            CK(cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, h->task_smem), "attr");
            CK(cudaFuncSetAttribute(ktd, cudaFuncAttributeMaxDynamicSharedMemorySize, h->task_smem), "attr");
            CK(cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, h->solo_smem), "attr");
            CK(cudaFuncSetAttribute(ksd, cudaFuncAttributeMaxDynamicSharedMemorySize, h->solo_smem), "attr");
            if (const char *ec = getenv("DTANS_TASK_CARVE")) {  // shared-memory carve-out preference (percent)
                const int pc = atoi(ec);
                CK(cudaFuncSetAttribute(kt, cudaFuncAttributePreferredSharedMemoryCarveout, pc), "carveout");
                CK(cudaFuncSetAttribute(ktd, cudaFuncAttributePreferredSharedMemoryCarveout, pc), "carveout");
                CK(cudaFuncSetAttribute(ks, cudaFuncAttributePreferredSharedMemoryCarveout, pc), "carveout");
                CK(cudaFuncSetAttribute(ksd, cudaFuncAttributePreferredSharedMemoryCarveout, pc), "carveout");
            }
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kt, dev::kTaskWarps * 32, h->task_smem), "occupancy");
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pers, ks, 256, h->solo_smem), "occupancy");
            return DTANS_OK;
        });
        if (rc) return rc;
        h->task_ctas = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * std::max(per, 1),
                                                                    ((int64_t)a.ntasks + dev::kTaskWarps - 1) / dev::kTaskWarps));
        h->solo_ctas = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * std::max(pers, 1),
                                                                    ((int64_t)a.nsolo + 255) / 256));
    }
    h->threads = dev::kMaxWarps * 32;  // all warps copy the tables; h->warps of them decode
    a.work_warps = h->warps;
    h->smem = sp.total;
    h->ctas = (int)std::max<int64_t>(1, std::min<int64_t>(sms, ((int64_t)h->chunks.size() + h->warps - 1) / h->warps));
    int per_sm = 0;
    int rc = with_kernel<V>(tb.dinline, h->pend, [&](auto kspmv, auto kspmv0, auto kdec, auto kscaled) -> int {
        CK(cudaFuncSetAttribute(kscaled, cudaFuncAttributeMaxDynamicSharedMemorySize, h->smem), "cudaFuncSetAttribute");
        CK(cudaFuncSetAttribute(kspmv, cudaFuncAttributeMaxDynamicSharedMemorySize, h->smem), "cudaFuncSetAttribute");
        CK(cudaFuncSetAttribute(kspmv0, cudaFuncAttributeMaxDynamicSharedMemorySize, h->smem), "cudaFuncSetAttribute");
        CK(cudaFuncSetAttribute(kdec, cudaFuncAttributeMaxDynamicSharedMemorySize, h->smem), "cudaFuncSetAttribute");
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kspmv, h->threads, h->smem), "occupancy");
        return DTANS_OK;
    });
    if (rc) return rc;
    if (per_sm < 1) return fail(DTANS_E_CUDA, "kernel does not fit on an SM");
    return DTANS_OK;
}

// x'[j] = x[map[j]] (symmetric reordering): one coalesced pass over x'
template <typename V>
__global__ void __launch_bounds__(256) permute_x_kernel(const V *__restrict__ x, const uint32_t *__restrict__ map,
                                                        V *__restrict__ xp, int64_t n)
{
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
        xp[j] = __ldg(x + __ldg(map + j));
}

// A long-slice kernel launched after its predecessor with programmatic
// dependent launch (kernels.cuh pdl_trigger/pdl_wait): it may start on the
// SMs the predecessor's finished CTAs free.
template <typename K>
void launch_chained(bool pdl, K kernel, int grid, int block, int smem, cudaStream_t st, const dev::KernelArgs &a)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, a);
}

template <typename V>
int launch(dtans_dev *h, const V *x, const V *y, V *out, const int64_t *row_start, int64_t *cols,
           void *vals, bool decode_only, cudaStream_t st, int64_t c_lo = -1, int64_t c_hi = -1,
           const double *sumsq_in = nullptr, double *sumsq_out = nullptr, double *sumsq_zero = nullptr,
           bool scaled = false)
{
    if (h->nslices == 0) return DTANS_OK;
    dev::KernelArgs a = h->base;
    if (c_lo >= 0) {  // chunk range (pipelined host path; static order, no long slices)
        a.chunk_lo = (uint32_t)c_lo;
        a.chunk_hi = (uint32_t)c_hi;
    }
    const int64_t nch = (int64_t)a.chunk_hi - (int64_t)a.chunk_lo;
    const int ctas = (int)std::max<int64_t>(1, std::min<int64_t>(h->sms, (nch + h->warps - 1) / h->warps));
    // solo kernel first, the task kernel beside it (PDL) taking tickets
    const bool solo_first = h->pdl != 0 && h->solo_first && a.nsolo > 0 && a.ntasks > 0 && c_lo < 0;
    a.task_dyn = solo_first ? 1 : 0;
    if (a.dynamic || a.task_dyn)
        CK(cudaMemsetAsync(a.work_counter, 0, 2 * sizeof(uint32_t), st), "reset work counters");
    if (h->d_col_map && !decode_only) {
        if (c_lo <= 0) {  // once per product (the pipelined host path gathers before its first chunk)
            const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)h->sms * 8, (h->cols + 255) / 256));
            permute_x_kernel<V><<<blocks, 256, 0, st>>>(x, h->d_col_map, (V *)h->d_xperm, h->cols);
            h->launches++;
        }
        x = (const V *)h->d_xperm;
    }
    a.x = x;
    a.y = y;
    a.out = out;
    a.row_start = row_start;
    a.dec_cols = cols;
    a.dec_vals = vals;
    a.sumsq_in = sumsq_in;
    a.sumsq_out = sumsq_out;
    a.sumsq_zero = sumsq_zero;
    if (nch > 0) {
        // the pending-products instantiation has no row-map lookup
        // PDL: the table copy overlaps the tail of a preceding main kernel
        // (the previous product on this stream); the kernel waits before it
        // touches x, y or the output.  Not on the pipelined host path.
        const bool pm = h->pdl_main && c_lo < 0;
        with_kernel<V>(h->dinline, h->pend && !h->d_row_map, [&](auto kspmv, auto kspmv0, auto kdec, auto kscaled) -> int {
            if (scaled)
                launch_chained(pm, kscaled, ctas, h->threads, h->smem, st, a);
            else if (decode_only)
                launch_chained(pm, kdec, ctas, h->threads, h->smem, st, a);
            else if (y != nullptr)
                launch_chained(pm, kspmv, ctas, h->threads, h->smem, st, a);
            else
                launch_chained(pm, kspmv0, ctas, h->threads, h->smem, st, a);
            return 0;
        });
        h->launches++;
    }
    if (scaled && nch <= 0 && sumsq_zero != nullptr)  // the main kernel zeroes it otherwise
        CK(cudaMemsetAsync(sumsq_zero, 0, sizeof(double), st), "zero sum of squares");
    if (a.nempty && c_lo < 0 && !decode_only) {
        const int eb = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)h->sms * 8, ((int64_t)a.nempty + 31) / 32));
        if (y != nullptr)
            launch_chained(h->pdl == 1 && nch > 0, dev::dtans_empty_kernel<V, true>, eb, 256, 0, st, a);
        else
            launch_chained(h->pdl == 1 && nch > 0, dev::dtans_empty_kernel<V, false>, eb, 256, 0, st, a);
        h->launches++;
    }
    if (a.nlong && c_lo < 0) {
        // the first long kernel overlaps the main kernel's tail only when the
        // main kernel ran in this call (it triggers its dependents early)
        const bool pdl = h->pdl != 0;
        bool chain = (h->pdl == 1 && nch > 0) || (pdl && a.nempty > 0 && !decode_only);
        with_long_kernels<V>(h->dinline, [&](auto kt, auto ktd, auto ks, auto ksd) -> int {
            if (solo_first) {
                launch_chained(chain, decode_only ? ksd : ks, h->solo_ctas, 256, h->solo_smem, st, a);
                launch_chained(true, decode_only ? ktd : kt, h->task_ctas, dev::kTaskWarps * 32, h->task_smem, st, a);
                chain = true;
                return 0;
            }
            if (a.ntasks) {
                launch_chained(chain, decode_only ? ktd : kt, h->task_ctas, dev::kTaskWarps * 32, h->task_smem, st, a);
                chain = pdl;
            }
            if (a.nsolo) {
                launch_chained(chain, decode_only ? ksd : ks, h->solo_ctas, 256, h->solo_smem, st, a);
                chain = pdl;
            }
            return 0;
        });
        h->launches += (a.ntasks ? 1 : 0) + (a.nsolo ? 1 : 0);
        const int nb = (int)(a.nlong_small_blocks + h->final_big);
        if (!decode_only && nb > 0) {
            if (y != nullptr)
                launch_chained(chain, dev::dtans_finalize_kernel<V, true>, nb, 256, 0, st, a);
            else
                launch_chained(chain, dev::dtans_finalize_kernel<V, false>, nb, 256, 0, st, a);
            h->launches += 1;
        }
    }
    CK(cudaGetLastError(), "kernel launch");
    return DTANS_OK;
}

// Worker threads over [0, n) in contiguous ranges (host-side assembly).
template <class F>
void parallel_for(size_t n, F &&f)
{
    const size_t nt = std::max<size_t>(1, std::min<size_t>({16, std::thread::hardware_concurrency(), (n + 63) / 64}));
    if (nt <= 1) {
        f(0, n);
        return;
    }
    std::vector<std::thread> th;
    for (size_t t = 0; t < nt; t++) th.emplace_back([&, t]() { f(n * t / nt, n * (t + 1) / nt); });
    for (auto &t : th) t.join();
}

// One chunk blob (kernels.cuh ChunkRec): slice metadata words, the slices'
// row_symbols, their stream words -- copied from the container arrays.
void assemble_chunk(const dtans_container_view *c, const dev::ChunkRec &r, const dev::ChunkRec *next, bool pads_ok,
                    uint32_t *p)
{
    const int64_t s0 = r.s0, k = r.kw & 0xFF;
    const uint64_t base = c->directory[s0];
    // the embedded record of the chunk the same warp buffer takes next
    if (next) {
        p[0] = (uint32_t)next->off;
        p[1] = (uint32_t)(next->off >> 32);
        p[2] = next->s0;
        p[3] = next->kw;
    } else {
        p[0] = p[1] = p[2] = p[3] = 0u;
    }
    p += 4;
    for (int64_t i = 0; i < k; i++) {
        // slice metadata word (kernels.cuh slice_meta)
        const int64_t sr0 = (s0 + i) * kSlice;
        uint32_t maxn = 0, minseg = 0xFFFFFFFFu;
        for (int64_t l = 0; l < kSlice; l++) {
            const uint32_t n = sr0 + l < c->rows ? c->row_symbols[sr0 + l] : 0u;
            maxn = std::max(maxn, n);
            minseg = std::min(minseg, (n + 7u) / 8u);
        }
        const uint32_t mseg = (maxn + 7u) / 8u;
        const uint32_t np = pads_ok && mseg > 0 ? (maxn - 8u * (mseg - 1u)) / 2u : 4u;
        p[i] = dev::slice_meta((uint32_t)(c->directory[s0 + i + 1] - base), mseg, minseg, np);
    }
    const uint32_t hw = dev::chunk_hdr_words((uint32_t)k) - 4u;
    for (uint32_t i = (uint32_t)k; i < hw; i++) p[i] = 0u;
    p += hw;
    const int64_t r0 = s0 * kSlice, r1 = std::min<int64_t>((s0 + k) * kSlice, c->rows);
    memcpy(p, c->row_symbols + r0, sizeof(uint32_t) * (size_t)(r1 - r0));
    for (int64_t i = r1 - r0; i < k * 32; i++) p[i] = 0u;
    p += k * 32;
    const uint64_t nw = c->directory[s0 + k] - base;
    memcpy(p, c->stream + base, sizeof(uint32_t) * (size_t)nw);
    for (uint64_t i = nw; i < ((nw + 3) & ~3ull); i++) p[i] = 0u;
}

// The GPU pre-pass of the long-slice index (kernels.cuh dtans_walk_kernel):
// one warp per long slice walks it once and writes the resume records into
// the device pool (whose masks the host plan already holds) and the task
// boundary cursors, which are copied back into the task lists here.
template <typename V>
int gpu_walk(dtans_dev *h, const TableBlock &tb, const SmemPlan &sp, const dtans_container_view *c, LongIndex &li,
             uint32_t *d_pool, int chunk)
{
    fill_args(h, tb, sp);
    const dev::KernelArgs &a = h->base;
    const size_t nparts = li.nparts, nl = li.slices.size();
    uint32_t *d_cur = nullptr;
    CK(cudaMalloc(&d_cur, sizeof(uint32_t) * (nparts + nl)), "cudaMalloc(walk cursors)");
    const int smem = (int)align_up((size_t)(a.off_img + a.table_bytes), 16);
    const int blocks = (int)std::max<size_t>(1, std::min<size_t>((size_t)h->sms * 8, (nl + 7) / 8));
    cudaError_t e = cudaSuccess;
    auto run = [&](auto k) {
        if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)) != cudaSuccess) return;
        k<<<blocks, 256, smem>>>(a, d_pool, d_cur, d_cur + nparts, (uint32_t)chunk);
        e = cudaGetLastError();
    };
    if (tb.dinline) run(dev::dtans_walk_kernel<V, true>);
    else run(dev::dtans_walk_kernel<V, false>);
    std::vector<uint32_t> cur(nparts + nl);
    if (e == cudaSuccess) e = cudaMemcpy(cur.data(), d_cur, sizeof(uint32_t) * cur.size(), cudaMemcpyDeviceToHost);
    cudaFree(d_cur);
    if (e != cudaSuccess) return cuda_fail(e, "checkpoint walk");
    unsigned int err = 0;
    CK(cudaMemcpy(&err, h->d_err, sizeof(err), cudaMemcpyDeviceToHost), "checkpoint walk status");
    if (err & 4u) return fail(DTANS_E_CUDA, "checkpoint walk: shared-memory layout check failed");
    // end cursor of every part: the next part's start in the same slice, or the slice's word count
    std::vector<uint32_t> end(nparts, 0);
    for (size_t i = 0; i < nl; i++) {
        const LongSlice &ls = li.slices[i];
        const uint32_t nw = (uint32_t)(c->directory[ls.slice + 1] - c->directory[ls.slice]);
        if (cur[nparts + i] != nw) return fail(DTANS_E_CORRUPT, "long slice consumed an unexpected number of words");
        for (uint32_t q = 0; q < ls.nparts; q++)
            end[ls.part_base + q] = q + 1 < ls.nparts ? cur[ls.part_base + q + 1] : nw;
    }
    for (LongTask &t : li.tasks) {
        t.cur0 = cur[t.part];
        t.cur1 = end[t.part];
    }
    for (SoloTask &t : li.solo) {
        t.cur0 = cur[t.part];
        t.cur1 = end[t.part];
    }
    return DTANS_OK;
}

// Pageable host buffers (the drop-in spmv's numpy arrays): copies go
// through two pinned staging buffers, filled / drained by worker threads
// while the other buffer's cudaMemcpyAsync runs -- the driver's own pageable
// path is several times slower.
struct HostStager {
    static constexpr size_t kCap = (size_t)16 << 20;
    void *buf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    bool ready = false;
    int init()
    {
        if (ready) return DTANS_OK;
        const unsigned hc = std::thread::hardware_concurrency();
        pool.start(hc > 1 ? (int)std::min(15u, hc - 1) : 0);
        for (int b = 0; b < 2; b++) {
            CK(cudaHostAlloc(&buf[b], kCap, cudaHostAllocDefault), "cudaHostAlloc staging");
            CK(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming), "event");
        }
        ready = true;
        return DTANS_OK;
    }
    // memcpy split over a persistent pool of worker threads (the calling
    // thread takes the first share); pageable destinations also take their
    // first-touch page faults in parallel
    struct Pool {
        std::vector<std::thread> th;
        std::mutex mu;
        std::condition_variable cv, done_cv;
        uint64_t gen = 0;
        int pending = 0;
        bool stop = false;
        char *dst = nullptr;
        const char *src = nullptr;
        size_t n = 0;
        int parts = 1;
        void run_part(int i)
        {
            const size_t lo = n * (size_t)i / (size_t)parts, hi = n * (size_t)(i + 1) / (size_t)parts;
            if (hi > lo) memcpy(dst + lo, src + lo, hi - lo);
        }
        void start(int workers)
        {
            parts = workers + 1;
            for (int w = 0; w < workers; w++)
                th.emplace_back([this, w]() {
                    uint64_t seen = 0;
                    for (;;) {
                        std::unique_lock<std::mutex> lk(mu);
                        cv.wait(lk, [&] { return stop || gen != seen; });
                        if (stop) return;
                        seen = gen;
                        lk.unlock();
                        run_part(w + 1);
                        lk.lock();
                        if (--pending == 0) done_cv.notify_one();
                    }
                });
        }
        void copy(char *d, const char *s, size_t len)
        {
            if (th.empty() || len < ((size_t)1 << 20)) {
                memcpy(d, s, len);
                return;
            }
            {
                std::lock_guard<std::mutex> lk(mu);
                dst = d;
                src = s;
                n = len;
                pending = (int)th.size();
                gen++;
            }
            cv.notify_all();
            run_part(0);
            std::unique_lock<std::mutex> lk(mu);
            done_cv.wait(lk, [&] { return pending == 0; });
        }
        ~Pool()
        {
            {
                std::lock_guard<std::mutex> lk(mu);
                stop = true;
            }
            cv.notify_all();
            for (auto &t : th) t.join();
        }
    } pool;
    void pcopy(char *dst, const char *src, size_t n) { pool.copy(dst, src, n); }
    int h2d(void *dst, const void *src, size_t n, cudaStream_t st)
    {
        int b = 0;
        for (size_t o = 0; o < n; o += kCap, b ^= 1) {
            const size_t len = std::min(kCap, n - o);
            CK(cudaEventSynchronize(ev[b]), "staging wait");
            pcopy((char *)buf[b], (const char *)src + o, len);
            CK(cudaMemcpyAsync((char *)dst + o, buf[b], len, cudaMemcpyHostToDevice, st), "staged H2D");
            CK(cudaEventRecord(ev[b], st), "event");
        }
        return DTANS_OK;
    }
    int d2h(void *dst, const void *src, size_t n, cudaStream_t st)
    {
        // piece i+1's copy is in flight while piece i is drained
        const size_t np = (n + kCap - 1) / kCap;
        for (size_t i = 0; i <= np; i++) {
            if (i < np) {
                const size_t o = i * kCap, len = std::min(kCap, n - o);
                CK(cudaEventSynchronize(ev[i & 1]), "staging wait");
                CK(cudaMemcpyAsync(buf[i & 1], (const char *)src + o, len, cudaMemcpyDeviceToHost, st), "staged D2H");
                CK(cudaEventRecord(ev[i & 1], st), "event");
            }
            if (i > 0) {
                const size_t q = i - 1, o = q * kCap, len = std::min(kCap, n - o);
                CK(cudaEventSynchronize(ev[q & 1]), "staging wait");
                pcopy((char *)dst + o, (const char *)buf[q & 1], len);
            }
        }
        return DTANS_OK;
    }
    ~HostStager()
    {
        for (int b = 0; b < 2; b++) {
            if (ev[b]) cudaEventDestroy(ev[b]);
            if (buf[b]) cudaFreeHost(buf[b]);
        }
    }
};

void free_stager(void *p) { delete (HostStager *)p; }

bool is_pageable(const void *p)
{
    if (!p) return false;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return at.type == cudaMemoryTypeUnregistered;
}

// Host->device copies through two pinned staging buffers on one stream:
// the host fills buffer b while buffer b^1's cudaMemcpyAsync is in flight.
struct PinnedUploader {
    static constexpr size_t kCap = (size_t)32 << 20;
    size_t cap = kCap;
    void *buf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    bool busy[2] = {false, false};
    int cur = 0;
    cudaStream_t st = nullptr;
    cudaError_t err = cudaSuccess;
    size_t bytes = 0;
    int64_t batches = 0;

    int init(int /*device*/)
    {
        // DTANS_UPLOAD_KB: staging buffer size (tests force many batches)
        if (const char *e = getenv("DTANS_UPLOAD_KB")) cap = std::max<size_t>(64, (size_t)atoll(e)) << 10;
        for (int b = 0; b < 2; b++) {
            if ((err = cudaHostAlloc(&buf[b], cap, cudaHostAllocDefault)) != cudaSuccess) return cuda_fail(err, "cudaHostAlloc");
            if ((err = cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming)) != cudaSuccess) return cuda_fail(err, "event");
        }
        if ((err = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)) != cudaSuccess) return cuda_fail(err, "stream");
        return DTANS_OK;
    }
    // the next free staging buffer (waits for its previous copy)
    void *acquire()
    {
        if (busy[cur]) {
            if ((err = cudaEventSynchronize(ev[cur])) != cudaSuccess) return nullptr;
            busy[cur] = false;
        }
        return buf[cur];
    }
    bool submit(void *dst, size_t n)
    {
        if ((err = cudaMemcpyAsync(dst, buf[cur], n, cudaMemcpyHostToDevice, st)) != cudaSuccess) return false;
        if ((err = cudaEventRecord(ev[cur], st)) != cudaSuccess) return false;
        busy[cur] = true;
        cur ^= 1;
        bytes += n;
        batches++;
        return true;
    }
    // a plain array (pageable or mmapped) through the staging buffers
    bool copy(void *dst, const void *src, size_t n)
    {
        const char *s = (const char *)src;
        char *d = (char *)dst;
        for (size_t o = 0; o < n; o += cap) {
            const size_t len = std::min(cap, n - o);
            char *b = (char *)acquire();
            if (!b) return false;
            parallel_for((len + 4095) / 4096, [&](size_t lo, size_t hi) {
                memcpy(b + lo * 4096, s + o + lo * 4096, std::min(len, hi * 4096) - lo * 4096);
            });
            if (!submit(d + o, len)) return false;
        }
        return true;
    }
    bool finish()
    {
        if (st && (err = cudaStreamSynchronize(st)) != cudaSuccess) return false;
        return true;
    }
    ~PinnedUploader()
    {
        if (st) {
            cudaStreamSynchronize(st);
            cudaStreamDestroy(st);
        }
        for (int b = 0; b < 2; b++) {
            if (ev[b]) cudaEventDestroy(ev[b]);
            if (buf[b]) cudaFreeHost(buf[b]);
        }
    }
};

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
    for (int64_t s = 0; s < nsl; s++)
        if (c->directory[s + 1] < c->directory[s]) return fail(DTANS_E_CORRUPT, "directory is not monotone");
    int max_optin = 0, sms = 0;
    CK(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device), "attr");
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device), "sm count");

    dtans_dev *h = new dtans_dev();
    h->device = device;
    h->sms = sms;
    h->rows = c->rows;
    h->cols = c->cols;
    h->nnz = c->nnz;
    h->nslices = nsl;
    h->nwords = c->nwords;
    h->precision = c->precision;
    const TableBlock tb = build_table_block(c->tables, c->precision);

    // per-slice cost (segments of the longest row) and the long-slice split
    const char *e1 = getenv("DTANS_LONG_SEG"), *e2 = getenv("DTANS_CHUNK");
    // chunked slices have max_nseg <= long_seg <= kMetaMaxNseg (slice_meta field)
    const int long_seg = std::min<int>(e1 ? atoi(e1) : 64, (int)dev::kMetaMaxNseg);
    // 24 segments per task (natural-order R-MAT: 8/12/16/20/24/28/32 gave
    // 1.622/1.592/1.626/1.663/1.577/1.618/1.648 ms -- non-monotonic, the
    // task/solo split shifts with it); rows-sorted plans use 48 (below)
    int chunk = e2 ? atoi(e2) : 24;
    const bool pads_ok = tb.nd > 0 && tb.nv > 0;
    std::vector<uint32_t> cost((size_t)nsl);
    for (int64_t s = 0; s < nsl; s++) {
        uint32_t m = 0;
        for (int64_t i = s * kSlice; i < std::min<int64_t>((s + 1) * kSlice, c->rows); i++)
            m = std::max(m, c->row_symbols[i]);
        cost[s] = (m + 7) / 8;
    }
    // staging ring: 2 buffers per warp (measured: larger chunks beat a
    // deeper ring; 32 warps x 2 chunks in flight cover the HBM latency)
    // DTANS_SMEM_KB caps the main kernel's shared memory (the rest of the
    // SM's 256 KB L1/shared array becomes L1 cache for the x gathers)
    const char *ek = getenv("DTANS_SMEM_KB");
    const int smem_cap = ek ? std::min(max_optin, atoi(ek) * 1024) : max_optin;
    // warps per CTA of the main kernel: 32, or fewer when the matrix has
    // fewer slices than a full grid has warps -- their staging buffers are
    // then larger, so small matrices' slices fit a buffer instead of going
    // to the long-slice kernels (DTANS_WARPS forces it)
    {
        const char *ew = getenv("DTANS_WARPS");
        int w = dev::kMaxWarps;
        if (ew) w = std::max(1, std::min(dev::kMaxWarps, atoi(ew)));
        else if (nsl < (int64_t)sms * dev::kMaxWarps)
            w = (int)std::max<int64_t>(4, std::min<int64_t>(dev::kMaxWarps, (nsl + sms - 1) / sms));
        h->warps = w;
    }
    SmemPlan sp = plan_smem(tb, smem_cap, dev::kMaxRing, h->warps);
    if (sp.bufb < 512) {
        delete h;
        return fail(DTANS_E_CUDA, "coding tables leave no shared memory for staging");
    }
    LongIndex li;
    {
        // a slice is long when even a one-slice chunk (chunk_words) overflows a buffer
        const uint64_t max_words = (uint64_t)(sp.bufb - 4 * (int)dev::chunk_hdr_words(1) - 128) / 4;
        // When rows are sorted by length (the skew toolkit's P*A) and most
        // nonzeros already sit in long slices, every non-empty slice goes to
        // the task kernel: one launch mixes the short, latency-bound slices
        // with the long, issue-bound tasks (R-MAT sorted: -4.5 %).  An
        // explicit DTANS_LONG_SEG wins.
        int seg_thr = long_seg;
        if (!e1) {
            uint64_t nnz_long = 0, nnz_all = 0;
            bool desc = true;
            for (int64_t s = 0; s < nsl; s++) {
                uint64_t z = 0;
                for (int64_t i = s * kSlice; i < std::min<int64_t>((s + 1) * kSlice, c->rows); i++)
                    z += c->row_symbols[i] / 2;
                nnz_all += z;
                const uint64_t words = ((c->directory[s + 1] + 3) & ~3ull) - (c->directory[s] & ~3ull);
                if (cost[s] > (uint32_t)long_seg || words > max_words) nnz_long += z;
                if (s > 0 && cost[s] > cost[s - 1]) desc = false;
            }
            if (desc && nnz_long * 2 >= nnz_all && nnz_all > 0) {
                seg_thr = 0;
                // sorted rows: neighbouring lanes end together, so longer
                // tasks lose little to idle lanes and halve the checkpoints
                // and partials (R-MAT sorted: 32 vs 16 segments -2.8 %, 48 another -1.2 %, 64 the same)
                if (!e2) chunk = 48;
            }
        }
        // the long-slice walk runs on the GPU (dtans_walk_kernel) unless
        // DTANS_GPU_WALK=0 (the multithreaded host walk)
        const char *eg = getenv("DTANS_GPU_WALK");
        h->host_walk = eg && atoi(eg) == 0;
        const int rc0 = build_long_index(c, seg_thr, max_words, std::max(1, chunk), h->host_walk, li);
        if (rc0) {
            delete h;
            return rc0;
        }
        h->base.ntasks = (uint32_t)li.tasks.size();
        h->base.nsolo = (uint32_t)li.solo.size();
        h->base.nlong = (uint32_t)li.slices.size();
        uint32_t small = 0, big = 0;
        while (small < li.slices.size() && li.slices[small].nparts >= 2 && li.slices[small].nparts <= 32) small++;
        while (small + big < li.slices.size() && li.slices[small + big].nparts > 32) big++;
        h->final_big = big;
        h->base.nlong_small = small;
        h->base.nlong_small_blocks = (small + 7) / 8;
        h->base.single_direct = 1;
        for (const LongSlice &ls : li.slices)
            if (ls.nparts > 1) h->split_slices.push_back(ls.slice);
        std::sort(h->split_slices.begin(), h->split_slices.end());
    }
    // chunk list over the slices the main kernel decodes
    {
        std::vector<uint8_t> is_long((size_t)nsl, 0);
        for (const LongSlice &ls : li.slices) is_long[ls.slice] = 1;
        // with long slices (no pipelined host path), all-empty slices go to
        // dtans_empty_kernel instead of the chunk list (DTANS_EMPTY=0: keep)
        std::vector<uint32_t> empty;
        const char *ee = getenv("DTANS_EMPTY");
        if (!li.slices.empty() && !(ee && atoi(ee) == 0)) {
            for (int64_t s = 0; s < nsl; s++) {
                if (is_long[s] || c->directory[s + 1] != c->directory[s]) continue;
                bool all0 = true;
                for (int64_t i = s * kSlice; i < std::min<int64_t>((s + 1) * kSlice, c->rows) && all0; i++)
                    all0 = c->row_symbols[i] == 0;
                if (all0) {
                    empty.push_back((uint32_t)s);
                    is_long[s] = 1;  // not in the chunk list
                }
            }
        }
        if (!empty.empty()) {
            cudaError_t e = cudaMalloc(&h->d_empty, sizeof(uint32_t) * empty.size());
            if (e == cudaSuccess)
                e = cudaMemcpy(h->d_empty, empty.data(), sizeof(uint32_t) * empty.size(), cudaMemcpyHostToDevice);
            if (e != cudaSuccess) {
                if (h->d_empty) cudaFree(h->d_empty);
                delete h;
                return fail(DTANS_E_NOMEM, "empty-slice list: %s", cudaGetErrorString(e));
            }
            h->base.empty_slices = h->d_empty;
            h->base.nempty = (uint32_t)empty.size();
        }
        double mean = 0;
        uint32_t mx = 0;
        for (int64_t s = 0; s < nsl; s++) {
            const uint32_t cs = is_long[s] ? 0 : cost[s];
            mean += cs;
            mx = std::max(mx, cs);
        }
        mean /= (double)std::max<int64_t>(nsl, 1);
        const char *ed = getenv("DTANS_DYNAMIC");
        const bool dyn = ed ? atoi(ed) != 0 : (mx > 4.0 * std::max(mean, 1.0));
        h->base.dynamic = dyn ? 1 : 0;
        bool sorted = true;
        for (int64_t s = 1; s < nsl && sorted; s++)
            sorted = (is_long[s] ? 0 : cost[s]) <= (is_long[s - 1] ? 0 : cost[s - 1]);
        const char *ek = getenv("DTANS_KCHUNK");
        // slices per chunk: aim at >= 4 chunks per warp, but at least 3 slices
        // once every warp has work (per-chunk overhead; a strong-scaling shard
        // of the Laplacian at N=8: -10 %), 1 for matrices smaller than the grid
        const int64_t grid_warps = (int64_t)sms * h->warps;
        const int64_t kcap = ek ? std::max(1, std::min(atoi(ek), dev::kMaxChunk))
                                : nsl < grid_warps ? 1
                                : std::max<int64_t>(3, std::min<int64_t>(dev::kMaxChunk, nsl / (grid_warps * 4)));
        uint64_t blob_words = 0;
        bool overflow = false;  // a chunk larger than a staging buffer (planner bug: fail loudly)
        auto push = [&](int64_t s0, int64_t k) {
            const uint64_t w = chunk_words(c->directory, s0, k);
            if (4 * w > (uint64_t)sp.bufb) overflow = true;
            h->chunks.push_back(dev::ChunkRec{blob_words, (uint32_t)s0, (uint32_t)k | (uint32_t)w << 8});
            blob_words += w;
        };

        if (dyn && !sorted) {
            // skewed, unsorted: single-slice chunks, longest first
            std::vector<uint32_t> order;
            for (int64_t s = 0; s < nsl; s++)
                if (!is_long[s]) order.push_back((uint32_t)s);
            std::stable_sort(order.begin(), order.end(), [&](uint32_t p, uint32_t q) { return cost[p] > cost[q]; });
            for (uint32_t s : order) push(s, 1);
        } else {
            int64_t s = 0;
            while (s < nsl) {
                if (is_long[s]) {
                    s++;
                    continue;
                }
                int64_t k = 1;
                while (k < kcap && s + k < nsl && !is_long[s + k] &&
                       chunk_bytes(c->directory, s, k + 1) <= (uint64_t)sp.bufb)
                    k++;
                push(s, k);
                s += k;
            }
        }
        h->blob_words = blob_words;
        if (overflow) {
            delete h;
            return fail(DTANS_E_PARAM, "internal: a chunk does not fit a staging buffer");
        }
        // static plans embed each chunk's successor in the same warp buffer
        // (chunk + 2 x the full grid's stride) in its blob
        h->base.embed_stride = dyn ? 0u : (uint32_t)(sms * h->warps);
        // the pending-products instantiation pays off where most staged
        // slices are hot up to a one-pair final segment (kernels.cuh
        // decode_range kPend, e.g. the 5-point Laplacian); elsewhere its
        // extra registers only cost (DTANS_PEND=0/1 forces it)
        int64_t staged = 0, pendable = 0;
        for (int64_t s = 0; s < nsl; s++) {
            if (is_long[s]) continue;
            staged++;
            uint32_t maxn = 0, minseg = 0xFFFFFFFFu;
            for (int64_t i = s * kSlice; i < (s + 1) * kSlice; i++) {
                const uint32_t n = i < c->rows ? c->row_symbols[i] : 0u;
                maxn = std::max(maxn, n);
                minseg = std::min(minseg, (n + 7u) / 8u);
            }
            const uint32_t mseg = (maxn + 7u) / 8u;
            if (pads_ok && mseg >= 2 && minseg == mseg && maxn - 8u * (mseg - 1u) <= 2u) pendable++;
        }
        if (const char *e = getenv("DTANS_PDL")) h->pdl = atoi(e);
        if (const char *e = getenv("DTANS_SOLO_FIRST")) h->solo_first = atoi(e) != 0;
        if (const char *e = getenv("DTANS_PDL_MAIN")) h->pdl_main = atoi(e) != 0;
        const char *ep = getenv("DTANS_PEND");
        h->pend = ep ? atoi(ep) != 0 : (staged > 0 && 2 * pendable >= staged);
    }

    // one allocation: [table image][chunk blobs][err][chunk records]
    //   + [row_symbols][directory][stream + pad] when long slices need them
    const bool need_raw = !li.tasks.empty() || !li.solo.empty();
    size_t off = 0;
    const size_t o_tb = off; off = align_up(off + sp.image.size() * 4, 256);
    const size_t o_bl = off; off = align_up(off + sizeof(uint32_t) * (size_t)std::max<uint64_t>(h->blob_words, 4), 256);
    const size_t o_er = off; off = align_up(off + 64, 256);
    const size_t o_ch = off; off = align_up(off + sizeof(dev::ChunkRec) * std::max<size_t>(h->chunks.size(), 1), 256);
    size_t o_rs = 0, o_di = 0, o_st = 0;
    if (need_raw) {
        o_rs = off; off = align_up(off + sizeof(uint32_t) * (size_t)std::max<int64_t>(c->rows, 1), 256);
        o_di = off; off = align_up(off + sizeof(uint64_t) * (size_t)(nsl + 1), 256);
        o_st = off; off = align_up(off + sizeof(uint32_t) * ((size_t)c->nwords + kRawStreamPad), 256);
    }
    cudaError_t e = cudaMalloc(&h->d_base, off);
    if (e != cudaSuccess) {
        delete h;
        return fail(DTANS_E_NOMEM, "cudaMalloc(%zu): %s", off, cudaGetErrorString(e));
    }
    h->d_bytes = off;
    char *b = (char *)h->d_base;
    h->d_tables = (uint32_t *)(b + o_tb);
    h->d_blob = (uint32_t *)(b + o_bl);
    h->d_err = (unsigned int *)(b + o_er);
    h->d_chunks = (dev::ChunkRec *)(b + o_ch);
    if (need_raw) {
        h->d_row_symbols = (uint32_t *)(b + o_rs);
        h->d_directory = (uint64_t *)(b + o_di);
        h->d_stream = (uint32_t *)(b + o_st);
    }
    int rc = DTANS_OK;
    auto cp = [&](void *dst, const void *src, size_t n) {
        if (rc == DTANS_OK && n) {
            cudaError_t ce = cudaMemcpy(dst, src, n, cudaMemcpyHostToDevice);
            if (ce != cudaSuccess) rc = cuda_fail(ce, "upload");
        }
    };
    auto zero = [&](void *dst, size_t n) {
        if (rc == DTANS_OK && n) {
            cudaError_t ce = cudaMemset(dst, 0, n);
            if (ce != cudaSuccess) rc = cuda_fail(ce, "memset");
        }
    };
    cp(h->d_tables, sp.image.data(), sp.image.size() * 4);
    {
        // Stream the chunk blobs to the device through pinned staging
        // buffers: worker threads assemble a batch of consecutive chunks
        // straight from the caller's arrays (possibly an mmapped CDTA file,
        // container.py:647-720) into one pinned buffer while the previous
        // batch's cudaMemcpyAsync runs; no full host copy of the container
        // is made.  Blobs are laid out in chunk order, so a batch is one
        // contiguous device range.
        const size_t nch = h->chunks.size();
        PinnedUploader up;
        if (rc == DTANS_OK) rc = up.init(device);
        size_t q = 0;
        while (rc == DTANS_OK && q < nch) {
            const uint64_t off0 = h->chunks[q].off;
            size_t qe = q;
            while (qe < nch && (h->chunks[qe].off + (h->chunks[qe].kw >> 8) - off0) * 4 <= up.cap) qe++;
            if (qe == q) {
                rc = fail(DTANS_E_PARAM, "chunk larger than the upload staging buffer");
                break;
            }
            const uint64_t words = h->chunks[qe - 1].off + (h->chunks[qe - 1].kw >> 8) - off0;
            uint32_t *dst = (uint32_t *)up.acquire();
            if (!dst) {
                rc = cuda_fail(up.err, "upload staging");
                break;
            }
            parallel_for(qe - q, [&](size_t lo, size_t hi) {
                for (size_t i = lo; i < hi; i++) {
                    const dev::ChunkRec &r = h->chunks[q + i];
                    const size_t nq = q + i + (size_t)dev::kMaxRing * h->base.embed_stride;
                    assemble_chunk(c, r, h->base.embed_stride && nq < nch ? &h->chunks[nq] : nullptr, pads_ok,
                                   dst + (r.off - off0));
                }
            });
            if (!up.submit(h->d_blob + off0, words * 4)) rc = cuda_fail(up.err, "upload chunk blobs");
            q = qe;
        }
        if (rc == DTANS_OK && need_raw) {
            // the long-slice kernels read the reference arrays directly
            if (!up.copy(h->d_row_symbols, c->row_symbols, sizeof(uint32_t) * (size_t)c->rows) ||
                !up.copy(h->d_directory, c->directory, sizeof(uint64_t) * (size_t)(nsl + 1)) ||
                !up.copy(h->d_stream, c->stream, sizeof(uint32_t) * (size_t)c->nwords))
                rc = cuda_fail(up.err, "upload raw arrays");
            zero(h->d_stream + c->nwords, sizeof(uint32_t) * kRawStreamPad);
        }
        if (rc == DTANS_OK && !up.finish()) rc = cuda_fail(up.err, "upload");
        h->upload_staged_bytes = up.bytes;
        h->upload_batches = up.batches;
    }
    zero(h->d_err, 64);
    cp(h->d_chunks, h->chunks.data(), sizeof(dev::ChunkRec) * h->chunks.size());
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
            // partial slots of solo tasks are written for one lane only
            zero(h->base.partials, pa_b);
            cp(lb + tb_b, li.pool.data(), li.pool.size() * 4);
            cp(lb + tb_b + pl_b, li.slices.data(), li.slices.size() * sizeof(LongSlice));
            if (rc == DTANS_OK && !h->host_walk) {
                h->base.nlong = (uint32_t)li.slices.size();
                rc = c->precision == 8 ? gpu_walk<double>(h, tb, sp, c, li, (uint32_t *)(lb + tb_b), std::max(1, chunk))
                                       : gpu_walk<float>(h, tb, sp, c, li, (uint32_t *)(lb + tb_b), std::max(1, chunk));
            }
            cp(lb, li.tasks.data(), li.tasks.size() * sizeof(LongTask));
            cp((void *)h->base.solo, li.solo.data(), li.solo.size() * sizeof(SoloTask));
        }
    }
    if (rc == DTANS_OK)
        rc = c->precision == 8 ? configure<double>(h, tb, sp) : configure<float>(h, tb, sp);
    if (rc != DTANS_OK) {
        cudaFree(h->d_base);
        if (h->d_long) cudaFree(h->d_long);
        delete h;
        return rc;
    }
    if (getenv("DTANS_VERBOSE"))
        fprintf(stderr,
                "[dtans] rows=%lld slices=%lld chunks=%zu nring=%d bufb=%d smem=%d dinline=%d rep_d=%d rep_v=%d "
                "nlong=%u ntasks=%u nsolo=%u dynamic=%d task_smem=%d\n",
                (long long)h->rows, (long long)nsl, h->chunks.size(), sp.nring, sp.bufb, h->smem, (int)tb.dinline,
                tb.rep_d, tb.rep_v, h->base.nlong, h->base.ntasks, h->base.nsolo, h->base.dynamic, h->task_smem);
    *out = h;
    return DTANS_OK;
}

extern "C" void dtans_free(dtans_dev *h)
{
    if (!h) return;
    cudaSetDevice(h->device);
    if (h->d_base) cudaFree(h->d_base);
    if (h->d_long) cudaFree(h->d_long);
    if (h->d_empty) cudaFree(h->d_empty);
    if (h->d_row_map) cudaFree(h->d_row_map);
    if (h->d_col_map) cudaFree(h->d_col_map);
    if (h->d_xperm) cudaFree(h->d_xperm);
    if (h->d_io) cudaFree(h->d_io);
    if (h->h_err) cudaFreeHost(h->h_err);
    for (int k = 0; k < kHostChunks; k++) {
        if (h->ev_in[k]) cudaEventDestroy(h->ev_in[k]);
        if (h->ev_done[k]) cudaEventDestroy(h->ev_done[k]);
    }
    free_stager(h->stager);
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
    if (warps_per_cta) *warps_per_cta = h->warps;
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

extern "C" int dtans_set_col_map(dtans_dev *h, const uint32_t *host_map)
{
    if (!h) return fail(DTANS_E_PARAM, "null handle");
    CK(cudaSetDevice(h->device), "cudaSetDevice");
    if (!host_map) {
        if (h->d_col_map) cudaFree(h->d_col_map);
        if (h->d_xperm) cudaFree(h->d_xperm);
        h->d_col_map = nullptr;
        h->d_xperm = nullptr;
        return DTANS_OK;
    }
    std::vector<uint8_t> seen((size_t)h->cols, 0);
    for (int64_t i = 0; i < h->cols; i++) {
        if (host_map[i] >= (uint64_t)h->cols || seen[host_map[i]])
            return fail(DTANS_E_PARAM, "col map must be a permutation of [0, cols)");
        seen[host_map[i]] = 1;
    }
    const size_t n = (size_t)std::max<int64_t>(h->cols, 1);
    if (!h->d_col_map) CK(cudaMalloc(&h->d_col_map, sizeof(uint32_t) * n), "cudaMalloc col map");
    if (!h->d_xperm) CK(cudaMalloc(&h->d_xperm, (size_t)h->precision * n), "cudaMalloc x scratch");
    CK(cudaMemcpy(h->d_col_map, host_map, sizeof(uint32_t) * (size_t)h->cols, cudaMemcpyHostToDevice),
       "upload col map");
    return DTANS_OK;
}

extern "C" int64_t dtans_launch_count(const dtans_dev *h) { return h ? h->launches : 0; }

extern "C" int64_t dtans_split_slices(const dtans_dev *h, uint32_t *out, int64_t cap)
{
    if (!h) return fail(DTANS_E_PARAM, "null handle");
    const int64_t n = (int64_t)h->split_slices.size();
    if (out)
        for (int64_t i = 0; i < std::min(n, cap); i++) out[i] = h->split_slices[(size_t)i];
    return n;
}

extern "C" int dtans_plan(const dtans_dev *h, dtans_plan_t *out)
{
    if (!h || !out) return fail(DTANS_E_PARAM, "null argument");
    *out = dtans_plan_t{};
    out->nchunks = (int64_t)h->chunks.size();
    for (const dev::ChunkRec &r : h->chunks) {
        out->chunk_slices_max = std::max<int64_t>(out->chunk_slices_max, r.kw & 0xFF);
        out->staged_slices += r.kw & 0xFF;
    }
    out->nlong = h->base.nlong;
    out->ntasks = h->base.ntasks;
    out->nsolo = h->base.nsolo;
    out->dynamic = h->base.dynamic;
    out->dinline = h->dinline ? 1 : 0;
    out->bufb = h->base.bufb;
    out->nring = h->base.nring;
    out->upload_bytes = (int64_t)h->upload_staged_bytes;
    out->upload_batches = h->upload_batches;
    out->pend = h->pend ? 1 : 0;
    out->nempty = h->base.nempty;
    return DTANS_OK;
}

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

extern "C" int dtans_spmv_scaled(dtans_dev *h, const void *x, void *out, const double *sumsq_in, double *sumsq_out,
                                 double *sumsq_zero, void *stream)
{
    if (!h) return fail(DTANS_E_PARAM, "null handle");
    CK(cudaSetDevice(h->device), "cudaSetDevice");
    if (h->precision == 8)
        return launch<double>(h, (const double *)x, nullptr, (double *)out, nullptr, nullptr, nullptr, false,
                              (cudaStream_t)stream, -1, -1, sumsq_in, sumsq_out, sumsq_zero, true);
    return launch<float>(h, (const float *)x, nullptr, (float *)out, nullptr, nullptr, nullptr, false,
                         (cudaStream_t)stream, -1, -1, sumsq_in, sumsq_out, sumsq_zero, true);
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
        if (err & 4u) return fail(DTANS_E_CUDA, "shared-memory window not 16 KB aligned at the slot tables");
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
    const int64_t nchunks = (int64_t)h->chunks.size();
    const char *eh = getenv("DTANS_HOST_STAGES");
    const int stages = std::max(1, std::min(kHostChunks, eh ? atoi(eh) : 8));
    // y/out ranges are contiguous only in natural row order (no row map)
    const bool chunked = h->base.nlong == 0 && !h->base.dynamic && nchunks >= 64 * stages && !h->d_row_map;
    if (!h->st_in) {
        CK(cudaStreamCreateWithFlags(&h->st_in, cudaStreamNonBlocking), "stream");
        CK(cudaStreamCreateWithFlags(&h->st_comp, cudaStreamNonBlocking), "stream");
        CK(cudaStreamCreateWithFlags(&h->st_out, cudaStreamNonBlocking), "stream");
        for (int k = 0; k < kHostChunks; k++) {
            CK(cudaEventCreateWithFlags(&h->ev_in[k], cudaEventDisableTiming), "event");
            CK(cudaEventCreateWithFlags(&h->ev_done[k], cudaEventDisableTiming), "event");
        }
    }
    if (is_pageable(x) || is_pageable(y) || is_pageable(out)) {
        // pageable buffers: staged copies in, one launch, staged copies out
        if (!h->stager) h->stager = new HostStager();
        HostStager *sg = (HostStager *)h->stager;
        // each buffer on its own: pinned ones are copied directly, pageable
        // ones through the staging buffers
        int rc = sg->init();
        auto h2d = [&](void *d, const void *hsrc, size_t n) -> int {
            if (!is_pageable(hsrc)) {
                CK(cudaMemcpyAsync(d, hsrc, n, cudaMemcpyHostToDevice, h->st_comp), "H2D");
                return DTANS_OK;
            }
            return sg->h2d(d, hsrc, n, h->st_comp);
        };
        if (!rc) rc = h2d(dx, x, es * (size_t)h->cols);
        if (!rc && y) rc = h2d(dy, y, es * (size_t)h->rows);
        if (!rc)
            rc = h->precision == 8
                     ? launch<double>(h, (const double *)dx, y ? (const double *)dy : nullptr, (double *)dout, nullptr,
                                      nullptr, nullptr, false, h->st_comp)
                     : launch<float>(h, (const float *)dx, y ? (const float *)dy : nullptr, (float *)dout, nullptr,
                                     nullptr, nullptr, false, h->st_comp);
        if (!rc) {
            if (is_pageable(out))
                rc = sg->d2h(out, dout, es * (size_t)h->rows, h->st_comp);
            else
                CK(cudaMemcpyAsync(out, dout, es * (size_t)h->rows, cudaMemcpyDeviceToHost, h->st_comp), "D2H");
        }
        if (rc) return rc;
        CK(cudaStreamSynchronize(h->st_comp), "synchronize");
        return dtans_check(h, h->st_comp);
    }
    const int nch = chunked ? stages : 1;
    CK(cudaMemcpyAsync(dx, x, es * (size_t)h->cols, cudaMemcpyHostToDevice, h->st_in), "H2D x");
    for (int k = 0; k < nch; k++) {
        // chunks [c0, c1) cover rows [r0, r1) (natural order when chunked);
        // the last two stages are short (3/32 and 1/32 of the chunks), so the
        // tail after the final H2D -- the last kernel and D2H -- is short
        auto bound = [&](int q) -> int64_t {
            if (nch < 4) return nchunks * q / nch;
            if (q >= nch) return nchunks;
            if (q == nch - 1) return nchunks - nchunks / 32;
            return (nchunks - nchunks / 8) * q / (nch - 2);  // q <= nch - 2
        };
        const int64_t c0 = bound(k), c1 = bound(k + 1);
        int64_t r0 = 0, r1 = h->rows;
        if (chunked) {
            r0 = (int64_t)h->chunks[c0].s0 * kSlice;
            const dev::ChunkRec &last = h->chunks[c1 - 1];
            r1 = std::min<int64_t>(((int64_t)last.s0 + (last.kw & 0xFF)) * kSlice, h->rows);
        }
        if (y && r1 > r0)
            CK(cudaMemcpyAsync(dy + es * r0, (const char *)y + es * r0, es * (size_t)(r1 - r0),
                               cudaMemcpyHostToDevice, h->st_in), "H2D y");
        CK(cudaEventRecord(h->ev_in[k], h->st_in), "event");
        CK(cudaStreamWaitEvent(h->st_comp, h->ev_in[k], 0), "wait");
        int rc;
        const int64_t lo = chunked ? c0 : -1, hi = chunked ? c1 : -1;
        if (h->precision == 8)
            rc = launch<double>(h, (const double *)dx, y ? (const double *)dy : nullptr, (double *)dout,
                                nullptr, nullptr, nullptr, false, h->st_comp, lo, hi);
        else
            rc = launch<float>(h, (const float *)dx, y ? (const float *)dy : nullptr, (float *)dout,
                               nullptr, nullptr, nullptr, false, h->st_comp, lo, hi);
        if (rc) return rc;
        CK(cudaEventRecord(h->ev_done[k], h->st_comp), "event");
        CK(cudaStreamWaitEvent(h->st_out, h->ev_done[k], 0), "wait");
        if (r1 > r0)
            CK(cudaMemcpyAsync((char *)out + es * r0, dout + es * r0, es * (size_t)(r1 - r0),
                               cudaMemcpyDeviceToHost, h->st_out), "D2H out");
    }
    // the error word rides the copy-out stream behind the last chunk (whose
    // kernel is the last on st_comp): one synchronize for the whole call
    if (!h->h_err) CK(cudaMallocHost(&h->h_err, sizeof(unsigned int)), "cudaMallocHost error word");
    CK(cudaMemcpyAsync(h->h_err, h->d_err, sizeof(unsigned int), cudaMemcpyDeviceToHost, h->st_out), "D2H error word");
    CK(cudaStreamSynchronize(h->st_out), "synchronize");
    if (*h->h_err) return dtans_check(h, h->st_comp);  // clears it and maps it to the error
    return DTANS_OK;
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
