// C ABI of libdtans.so: device upload, fused SpMV / decode launches.
// Declarations and reference citations: include/dtans.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

#include "common.h"
#include "kernels.cuh"

using namespace dtans;

struct dtans_dev {
    int device = 0;
    int64_t rows = 0, cols = 0, nnz = 0, nslices = 0, nwords = 0;
    int32_t precision = 8;
    void *d_base = nullptr;     // single allocation for all container arrays
    size_t d_bytes = 0;
    uint2 *d_dtab = nullptr;
    void *d_vtab = nullptr;
    uint32_t *d_row_symbols = nullptr;
    uint64_t *d_directory = nullptr;
    uint32_t *d_stream = nullptr;
    unsigned int *d_err = nullptr;
    // staging buffers for the host-pointer entry point
    void *d_io = nullptr;
    size_t io_bytes = 0;
    int ctas = 0, threads = 512, smem = 0;
    int64_t launches = 0;
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

template <typename V>
int configure(dtans_dev *h)
{
    using Entry = typename dev::ValueTraits<V>::Entry;
    h->smem = (int)(dev::kSlots * (sizeof(uint2) + sizeof(Entry)));
    CK(cudaFuncSetAttribute(dev::dtans_spmv_kernel<V>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            h->smem),
       "cudaFuncSetAttribute");
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dev::dtans_spmv_kernel<V>, h->threads,
                                                     h->smem),
       "occupancy");
    if (per_sm < 1) return fail(DTANS_E_CUDA, "kernel does not fit on an SM");
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device), "sm count");
    const int64_t warps_needed = h->nslices;
    const int64_t ctas_needed = (warps_needed + h->threads / 32 - 1) / (h->threads / 32);
    h->ctas = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * per_sm, ctas_needed));
    return DTANS_OK;
}

template <typename V>
int launch(dtans_dev *h, const V *x, const V *y, V *out, const int64_t *row_start, int64_t *cols,
           void *vals, int decode_only, cudaStream_t st)
{
    if (h->nslices == 0) return DTANS_OK;
    dev::KernelArgs a;
    a.dtab = h->d_dtab;
    a.vtab = h->d_vtab;
    a.row_symbols = h->d_row_symbols;
    a.directory = h->d_directory;
    a.stream = h->d_stream;
    a.rows = h->rows;
    a.cols = h->cols;
    a.nslices = h->nslices;
    a.nwords = h->nwords;
    a.x = x;
    a.y = y;
    a.out = out;
    a.row_start = row_start;
    a.dec_cols = cols;
    a.dec_vals = vals;
    a.err = h->d_err;
    a.decode_only = decode_only;
    dev::dtans_spmv_kernel<V><<<h->ctas, h->threads, h->smem, st>>>(a);
    h->launches++;
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

    // re-laid-out slot tables (see kernels.cuh for the entry formats)
    const int rec = c->precision == 8 ? 16 : 12;
    const size_t vent = c->precision == 8 ? 16 : 8;
    std::vector<uint2> dt(kK);
    std::vector<uint32_t> vt(kK * vent / 4, 0);
    const uint64_t vsent = c->precision == 8 ? ~0ull : 0xFFFFFFFFull;
    for (int j = 0; j < kK; j++) {
        const uint8_t *r = c->tables + (size_t)j * rec;
        uint64_t vs = 0;
        uint32_t ds = 0;
        if (c->precision == 8) {
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
        const uint32_t desc = ds == (uint32_t)kDeltaSentinel;
        const uint32_t vesc = vs == vsent;
        dt[j].x = desc ? 0u : ds;
        dt[j].y = (uint32_t)r[0] | ((uint32_t)r[1] << 8) | (desc << 16);
        const uint32_t vmeta = (uint32_t)r[2] | ((uint32_t)r[3] << 8) | (vesc << 16);
        if (c->precision == 8) {
            const uint64_t v = vesc ? 0 : vs;
            vt[4 * j + 0] = (uint32_t)v;
            vt[4 * j + 1] = (uint32_t)(v >> 32);
            vt[4 * j + 2] = vmeta;
        } else {
            vt[2 * j + 0] = vesc ? 0u : (uint32_t)vs;
            vt[2 * j + 1] = vmeta;
        }
    }
    // one allocation: [dtab][vtab][row_symbols][directory][stream + pad][err]
    size_t off = 0;
    const size_t o_dt = off; off = align_up(off + kK * sizeof(uint2), 256);
    const size_t o_vt = off; off = align_up(off + kK * vent, 256);
    const size_t o_rs = off; off = align_up(off + sizeof(uint32_t) * (size_t)std::max<int64_t>(c->rows, 1), 256);
    const size_t o_di = off; off = align_up(off + sizeof(uint64_t) * (size_t)(nsl + 1), 256);
    const size_t o_st = off; off = align_up(off + sizeof(uint32_t) * (size_t)c->nwords + 64, 256);
    const size_t o_er = off; off = align_up(off + 16, 256);
    cudaError_t e = cudaMalloc(&h->d_base, off);
    if (e != cudaSuccess) {
        delete h;
        return fail(DTANS_E_NOMEM, "cudaMalloc(%zu): %s", off, cudaGetErrorString(e));
    }
    h->d_bytes = off;
    char *b = (char *)h->d_base;
    h->d_dtab = (uint2 *)(b + o_dt);
    h->d_vtab = b + o_vt;
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
    cp(h->d_dtab, dt.data(), kK * sizeof(uint2));
    cp(h->d_vtab, vt.data(), kK * vent);
    cp(h->d_row_symbols, c->row_symbols, sizeof(uint32_t) * (size_t)c->rows);
    cp(h->d_directory, c->directory, sizeof(uint64_t) * (size_t)(nsl + 1));
    cp(h->d_stream, c->stream, sizeof(uint32_t) * (size_t)c->nwords);
    if (rc == DTANS_OK) {
        cudaError_t ce = cudaMemset(h->d_stream + c->nwords, 0, 64);
        if (ce == cudaSuccess) ce = cudaMemset(h->d_err, 0, 16);
        if (ce != cudaSuccess) rc = cuda_fail(ce, "memset");
    }
    if (rc == DTANS_OK) rc = c->precision == 8 ? configure<double>(h) : configure<float>(h);
    if (rc != DTANS_OK) {
        cudaFree(h->d_base);
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
    if (h->d_io) cudaFree(h->d_io);
    delete h;
}

extern "C" int dtans_info(const dtans_dev *h, int64_t *device_bytes, int32_t *ctas,
                          int32_t *warps_per_cta, int32_t *smem_bytes)
{
    if (!h) return fail(DTANS_E_PARAM, "null handle");
    if (device_bytes) *device_bytes = (int64_t)h->d_bytes;
    if (ctas) *ctas = h->ctas;
    if (warps_per_cta) *warps_per_cta = h->threads / 32;
    if (smem_bytes) *smem_bytes = h->smem;
    return DTANS_OK;
}

extern "C" int64_t dtans_launch_count(const dtans_dev *h) { return h ? h->launches : 0; }

extern "C" int dtans_spmv_f64(dtans_dev *h, const double *x, const double *y, double *out,
                              void *stream)
{
    if (!h) return fail(DTANS_E_PARAM, "null handle");
    if (h->precision != 8) return fail(DTANS_E_PARAM, "container precision is f32");
    CK(cudaSetDevice(h->device), "cudaSetDevice");
    return launch<double>(h, x, y, out, nullptr, nullptr, nullptr, 0, (cudaStream_t)stream);
}

extern "C" int dtans_spmv_f32(dtans_dev *h, const float *x, const float *y, float *out,
                              void *stream)
{
    if (!h) return fail(DTANS_E_PARAM, "null handle");
    if (h->precision != 4) return fail(DTANS_E_PARAM, "container precision is f64");
    CK(cudaSetDevice(h->device), "cudaSetDevice");
    return launch<float>(h, x, y, out, nullptr, nullptr, nullptr, 0, (cudaStream_t)stream);
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
    cudaStream_t st = nullptr;
    CK(cudaMemcpyAsync(dx, x, es * (size_t)h->cols, cudaMemcpyHostToDevice, st), "H2D x");
    if (y) CK(cudaMemcpyAsync(dy, y, es * (size_t)h->rows, cudaMemcpyHostToDevice, st), "H2D y");
    int rc;
    if (h->precision == 8)
        rc = launch<double>(h, (const double *)dx, y ? (const double *)dy : nullptr, (double *)dout,
                            nullptr, nullptr, nullptr, 0, st);
    else
        rc = launch<float>(h, (const float *)dx, y ? (const float *)dy : nullptr, (float *)dout,
                           nullptr, nullptr, nullptr, 0, st);
    if (rc) return rc;
    CK(cudaMemcpyAsync(out, dout, es * (size_t)h->rows, cudaMemcpyDeviceToHost, st), "D2H out");
    return dtans_check(h, st);
}

extern "C" int dtans_decode(dtans_dev *h, const int64_t *row_start, int64_t *cols, void *valbits,
                            void *stream)
{
    if (!h) return fail(DTANS_E_PARAM, "null handle");
    CK(cudaSetDevice(h->device), "cudaSetDevice");
    if (h->precision == 8)
        return launch<double>(h, nullptr, nullptr, nullptr, row_start, cols, valbits, 1,
                              (cudaStream_t)stream);
    return launch<float>(h, nullptr, nullptr, nullptr, row_start, cols, valbits, 1,
                         (cudaStream_t)stream);
}
