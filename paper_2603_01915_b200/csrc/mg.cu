// Multi-GPU power iteration through NCCL (SURVEY §8b "dtans_mg_init /
// dtans_mg_power_iteration", §8e): one process per GPU, each holding a
// contiguous row shard of the matrix as its own dtans_dev handle (a slice
// range is itself a valid container, distributed.shard).  Per iteration:
//   1. the fused scaled SpMV of the local rows (dtans_spmv_scaled: y_k =
//      (A_local x_k) / ||y_{k-1}||, with sum(y_k^2) accumulated in its
//      epilogue);
//   2. ncclAllReduce of that one f64;
//   3. the all-gather of y_k into the next full-length x as grouped
//      ncclBroadcasts straight into each shard's row offset (shards are
//      unequal, so no padding and no compaction pass).
// All on one stream, so NCCL over NVLink/NVSwitch runs behind the kernel
// without host round trips.  NCCL is loaded at run time (dlopen of
// libnccl.so.2: the one torch already loaded, or the system one), so the
// library has no link-time NCCL dependency and the single-GPU entry points
// never need it.
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "common.h"

namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
};

const NcclApi &nccl()
{
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) return;
        auto sym = [&](auto &fp, const char *name) {
            fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(lib, name));
            return fp != nullptr;
        };
        api.ok = sym(api.GetUniqueId, "ncclGetUniqueId") && sym(api.CommInitRank, "ncclCommInitRank") &&
                 sym(api.CommDestroy, "ncclCommDestroy") && sym(api.AllReduce, "ncclAllReduce") &&
                 sym(api.Broadcast, "ncclBroadcast") && sym(api.GroupStart, "ncclGroupStart") &&
                 sym(api.GroupEnd, "ncclGroupEnd") && sym(api.GetErrorString, "ncclGetErrorString");
    });
    return api;
}

int nccl_fail(ncclResult_t r, const char *what)
{
    return dtans::fail(DTANS_E_CUDA, "%s: %s", what, nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error");
}

#define NK(call, what)                                   \
    do {                                                 \
        const ncclResult_t r_ = (call);                  \
        if (r_ != ncclSuccess) return nccl_fail(r_, what); \
    } while (0)
#define CKM(call, what)                                                                      \
    do {                                                                                     \
        const cudaError_t e_ = (call);                                                       \
        if (e_ != cudaSuccess) return dtans::fail(DTANS_E_CUDA, "%s: %s", what, cudaGetErrorString(e_)); \
    } while (0)

// x_out = y / sqrt(S) in the vector precision (torch: x / sqrt(S).to(dtype)).
template <typename V>
__global__ void normalize_kernel(const V *__restrict__ y, V *__restrict__ x, const double *S, int64_t n)
{
    const V norm = (V)__dsqrt_rn(*S);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = y[i] / norm;
}

}  // namespace

struct dtans_mg {
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0, device = 0;
    void *buf = nullptr;  // iteration scratch, kept across calls
    size_t bytes = 0;
};

extern "C" int dtans_mg_unique_id(uint8_t *id)
{
    if (!id) return dtans::fail(DTANS_E_PARAM, "null argument");
    if (!nccl().ok) return dtans::fail(DTANS_E_NODEVICE, "libnccl.so.2 could not be loaded");
    ncclUniqueId u;
    NK(nccl().GetUniqueId(&u), "ncclGetUniqueId");
    memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
    return DTANS_OK;
}

extern "C" int dtans_mg_init(const uint8_t *id, int nranks, int rank, int device, dtans_mg **out)
{
    if (!id || !out) return dtans::fail(DTANS_E_PARAM, "null argument");
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks) return dtans::fail(DTANS_E_PARAM, "bad rank %d of %d", rank, nranks);
    if (!nccl().ok) return dtans::fail(DTANS_E_NODEVICE, "libnccl.so.2 could not be loaded");
    CKM(cudaSetDevice(device), "cudaSetDevice");
    ncclUniqueId u;
    memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
    dtans_mg *g = new dtans_mg();
    g->nranks = nranks;
    g->rank = rank;
    g->device = device;
    const ncclResult_t r = nccl().CommInitRank(&g->comm, nranks, u, rank);
    if (r != ncclSuccess) {
        delete g;
        return nccl_fail(r, "ncclCommInitRank");
    }
    *out = g;
    return DTANS_OK;
}

extern "C" void dtans_mg_free(dtans_mg *g)
{
    if (!g) return;
    if (g->comm && nccl().ok) nccl().CommDestroy(g->comm);
    if (g->buf) cudaFree(g->buf);
    delete g;
}

extern "C" int dtans_mg_power_iteration(dtans_mg *g, dtans_dev *h, const int64_t *row_off, void *x, int iters,
                                        double *lambda_out, void *stream)
{
    if (!g || !h || !row_off || !x || !lambda_out) return dtans::fail(DTANS_E_PARAM, "null argument");
    int64_t rows = 0, cols = 0;
    int32_t prec = 8;
    dtans::dev_shape(h, &rows, &cols, &prec);
    const int64_t n = row_off[g->nranks];
    if (row_off[0] != 0 || cols != n || row_off[g->rank + 1] - row_off[g->rank] != rows)
        return dtans::fail(DTANS_E_PARAM, "the shard must hold rows [row_off[rank], row_off[rank+1]) of a square n x n matrix");
    for (int r = 0; r < g->nranks; r++)
        if (row_off[r + 1] < row_off[r]) return dtans::fail(DTANS_E_PARAM, "row_off must be nondecreasing");
    *lambda_out = NAN;
    if (iters <= 0) return DTANS_OK;
    CKM(cudaSetDevice(g->device), "cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    const size_t es = (size_t)prec;
    const ncclDataType_t dt = prec == 8 ? ncclFloat64 : ncclFloat32;
    // [S: 3 f64][xb: n].  The local rows of y_k are written straight into
    // their place in the next x, and broadcast from there in place.
    const size_t ob_x = 256, need = ob_x + es * (size_t)n;
    if (g->bytes < need) {
        if (g->buf) cudaFree(g->buf);
        g->buf = nullptr;
        g->bytes = 0;
        CKM(cudaMalloc(&g->buf, need), "cudaMalloc");
        g->bytes = need;
    }
    char *buf = (char *)g->buf;
    double *S = (double *)buf;
    void *xs[2] = {x, buf + ob_x};
    int status = DTANS_OK;
    auto run = [&]() -> int {
        CKM(cudaMemsetAsync(S, 0, 3 * sizeof(double), st), "memset");
        for (int k = 0; k < iters; k++) {
            void *xc = xs[k & 1], *xn = xs[(k + 1) & 1];
            void *y = (char *)xn + es * (size_t)row_off[g->rank];
            const int r = dtans_spmv_scaled(h, xc, y, k ? S + (k - 1) % 3 : nullptr, S + k % 3, S + (k + 1) % 3, st);
            if (r) return r;
            if (g->nranks == 1) continue;  // one shard: y_k is the next x already
            NK(nccl().AllReduce(S + k % 3, S + k % 3, 1, ncclFloat64, ncclSum, g->comm, st), "ncclAllReduce");
            NK(nccl().GroupStart(), "ncclGroupStart");
            for (int q = 0; q < g->nranks; q++) {
                const size_t cnt = (size_t)(row_off[q + 1] - row_off[q]);
                if (cnt == 0) continue;
                char *seg = (char *)xn + es * (size_t)row_off[q];
                NK(nccl().Broadcast(seg, seg, cnt, dt, q, g->comm, st), "ncclBroadcast");
            }
            NK(nccl().GroupEnd(), "ncclGroupEnd");
        }
        // x_iters = y_last / ||y_last|| into the caller's buffer
        const void *ylast = xs[iters & 1];
        const double *Sl = S + (iters - 1) % 3;
        const int blocks = (int)std::min<int64_t>(1184, (n + 255) / 256 + 1);
        if (prec == 8) normalize_kernel<double><<<blocks, 256, 0, st>>>((const double *)ylast, (double *)x, Sl, n);
        else normalize_kernel<float><<<blocks, 256, 0, st>>>((const float *)ylast, (float *)x, Sl, n);
        CKM(cudaGetLastError(), "normalize");
        double s = 0.0;
        CKM(cudaMemcpyAsync(&s, Sl, sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
        CKM(cudaStreamSynchronize(st), "synchronize");
        *lambda_out = std::sqrt(s);
        return DTANS_OK;
    };
    status = run();
    if (status == DTANS_OK) status = dtans_check(h, stream);
    return status;
}
