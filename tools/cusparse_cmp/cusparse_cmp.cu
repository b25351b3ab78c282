// cuSPARSE SpMV comparator: y = A x + y with the library's
// CSR (ALG1, ALG2), COO and sliced-ELL (slice 32) kernels on device arrays,
// timed with CUDA events.  A separate library (libcusparse_cmp.so): the
// product (libdtans.so) never links cuSPARSE; bench.py loads this one only to
// print comparator numbers next to the dtANS kernel.
#include <cuda_runtime.h>
#include <cusparse.h>

#include <cstdint>
#include <cstdio>

namespace {
thread_local char g_err[256] = "";
int fail(const char *what, int code)
{
    snprintf(g_err, sizeof(g_err), "%s failed (%d)", what, code);
    return 1;
}
}  // namespace

#define CSP(call)                                               \
    do {                                                        \
        const cusparseStatus_t s_ = (call);                     \
        if (s_ != CUSPARSE_STATUS_SUCCESS) { rc = fail(#call, (int)s_); goto done; } \
    } while (0)
#define CUD(call)                                               \
    do {                                                        \
        const cudaError_t e_ = (call);                          \
        if (e_ != cudaSuccess) { rc = fail(#call, (int)e_); goto done; } \
    } while (0)

extern "C" const char *cmp_last_error(void) { return g_err; }

// fmt: 0 = CSR ALG1, 1 = CSR ALG2, 2 = COO, 3 = SELL (slice 32).
//   CSR:  a0 = row offsets (rows+1), a1 = columns (nnz), a2 = values
//   COO:  a0 = row indices (nnz),    a1 = columns,        a2 = values
//   SELL: a0 = slice offsets (nslices+1), a1 = columns (sell_size, -1 = pad), a2 = values
// Index arrays are int32 (ibits 32: the 4-byte indices of the CSR byte
// model, reference sparse.py:185-198) or int64 (ibits 64).  prec 8 / 4.  Runs `warmup` then `iters` products on the legacy stream and
// writes the mean milliseconds per product.
extern "C" int cmp_spmv_time(int fmt, int64_t rows, int64_t cols, int64_t nnz, void *a0, void *a1, void *a2,
                             int64_t sell_size, int prec, int ibits, const void *x, void *y, int warmup,
                             int iters, float *ms_out)
{
    int rc = 0;
    cusparseHandle_t h = nullptr;
    cusparseSpMatDescr_t A = nullptr;
    cusparseDnVecDescr_t vx = nullptr, vy = nullptr;
    void *work = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    const cudaDataType dt = prec == 8 ? CUDA_R_64F : CUDA_R_32F;
    const double one_d = 1.0;
    const float one_f = 1.0f;
    const void *alpha = prec == 8 ? (const void *)&one_d : (const void *)&one_f;
    cusparseSpMVAlg_t alg = CUSPARSE_SPMV_ALG_DEFAULT;
    size_t wb = 0;
    float ms = 0.f;
    const cusparseIndexType_t it = ibits == 32 ? CUSPARSE_INDEX_32I : CUSPARSE_INDEX_64I;
    CSP(cusparseCreate(&h));
    switch (fmt) {
    case 0:
    case 1:
        CSP(cusparseCreateCsr(&A, rows, cols, nnz, a0, a1, a2, it, it,
                              CUSPARSE_INDEX_BASE_ZERO, dt));
        alg = fmt == 0 ? CUSPARSE_SPMV_CSR_ALG1 : CUSPARSE_SPMV_CSR_ALG2;
        break;
    case 2:
        CSP(cusparseCreateCoo(&A, rows, cols, nnz, a0, a1, a2, it, CUSPARSE_INDEX_BASE_ZERO, dt));
        alg = CUSPARSE_SPMV_COO_ALG1;
        break;
    case 3:
        CSP(cusparseCreateSlicedEll(&A, rows, cols, nnz, sell_size, 32, a0, a1, a2, it, it,
                                    CUSPARSE_INDEX_BASE_ZERO, dt));
        alg = CUSPARSE_SPMV_SELL_ALG1;
        break;
    default:
        rc = fail("format", fmt);
        goto done;
    }
    CSP(cusparseCreateDnVec(&vx, cols, (void *)x, dt));
    CSP(cusparseCreateDnVec(&vy, rows, y, dt));
    CSP(cusparseSpMV_bufferSize(h, CUSPARSE_OPERATION_NON_TRANSPOSE, alpha, A, vx, alpha, vy, dt, alg, &wb));
    if (wb) CUD(cudaMalloc(&work, wb));
    CUD(cudaEventCreate(&e0));
    CUD(cudaEventCreate(&e1));
    for (int i = 0; i < warmup; i++)
        CSP(cusparseSpMV(h, CUSPARSE_OPERATION_NON_TRANSPOSE, alpha, A, vx, alpha, vy, dt, alg, work));
    CUD(cudaDeviceSynchronize());
    CUD(cudaEventRecord(e0, 0));
    for (int i = 0; i < iters; i++)
        CSP(cusparseSpMV(h, CUSPARSE_OPERATION_NON_TRANSPOSE, alpha, A, vx, alpha, vy, dt, alg, work));
    CUD(cudaEventRecord(e1, 0));
    CUD(cudaEventSynchronize(e1));
    CUD(cudaEventElapsedTime(&ms, e0, e1));
    *ms_out = ms / (float)(iters > 0 ? iters : 1);
done:
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (work) cudaFree(work);
    if (vx) cusparseDestroyDnVec(vx);
    if (vy) cusparseDestroyDnVec(vy);
    if (A) cusparseDestroySpMat(A);
    if (h) cusparseDestroy(h);
    return rc;
}
