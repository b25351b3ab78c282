/*
 * dtans.h — the C ABI of libdtans.so (B200-native CSR-dtANS SpMV).
 *
 * The reference (/root/reference/pkg/src/csrdtans) is a pure-Python package
 * with no FFI; its plugin surface for this path is the Python API
 *   encode_matrix  container.py:126-204
 *   spmv           container.py:554-596
 *   decode_matrix  container.py:524-531
 *   quantize       entropy.py:223-321
 * Each entry point below replaces the body of one of those functions; the
 * Python package paper_2603_01915_b200 binds them with ctypes exactly as a
 * maintainer of the reference would.
 *
 * Plain pointers and sizes only; no torch types.  All functions return a
 * dtans_status; on failure dtans_last_error() holds a message (per thread).
 * Device pointers are CUDA global-memory pointers on the handle's device;
 * "stream" is a cudaStream_t passed as void* (NULL = legacy default stream).
 */
#ifndef DTANS_H
#define DTANS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    DTANS_OK = 0,
    DTANS_E_PARAM = 1,    /* -> ParameterError (entropy.py:18)            */
    DTANS_E_CODING = 2,   /* -> CodingError    (entropy.py:22)            */
    DTANS_E_CORRUPT = 3,  /* -> CorruptStream  (entropy.py:26)            */
    DTANS_E_CUDA = 4,     /* CUDA runtime failure                         */
    DTANS_E_NOMEM = 5,    /* host or device allocation failed             */
    DTANS_E_NODEVICE = 6  /* no CUDA device: the product has no CPU path  */
} dtans_status;

/* Message for the last failure on the calling thread ("" if none). */
const char *dtans_last_error(void);

/* ABI version (bumped when a struct layout changes). */
int dtans_abi_version(void);

/* ------------------------------------------------------------------ */
/* Encoder (host, C++17, multithreaded).  Byte-identical to the
 * reference encode_matrix (container.py:126-204). */

typedef struct {
    int64_t rows, cols, nnz;
    const int64_t *row_start; /* rows + 1 */
    const int64_t *col_idx;   /* nnz, strictly ascending per row */
    const void *values;       /* nnz values already in the container precision */
    int32_t precision;        /* 4 (f32) or 8 (f64) */
} dtans_csr_view;

typedef struct {
    int32_t k_log2;              /* 12 (K = 4096)                           */
    int32_t m_log2;              /* <= 8 (M <= 256)                         */
    const uint32_t *perm_delta;  /* K-entry slot permutation or NULL       */
    const uint32_t *perm_value;  /* (numpy default_rng(seed).permutation)  */
    int32_t threads;             /* 0 = all hardware threads               */
} dtans_encode_opts;

/* Encoder output, allocated by the library; release with
 * dtans_encoded_free.  tables holds K serialized slot records in the
 * reference layout (container.py:604-609): 16 B (f64) / 12 B (f32). */
typedef struct {
    int64_t rows, cols, nnz, nslices, nwords;
    int32_t precision, rec_size;
    uint8_t *tables;       /* K * rec_size bytes */
    uint32_t *row_symbols; /* rows              */
    uint64_t *directory;   /* nslices + 1       */
    uint32_t *stream;      /* nwords            */
} dtans_encoded;

/* Replaces encode_matrix (container.py:126-204): validation (sparse.py:76-91),
 * distributions (container.py:112-114), quantize (entropy.py:223-321) x2,
 * build_tables (entropy.py:404-436) x2, per-row dtans_encode
 * (codec.py:296-368), interleave_warp (container.py:283-317). */
int dtans_encode(const dtans_csr_view *m, const dtans_encode_opts *opts,
                 dtans_encoded *out);
void dtans_encoded_free(dtans_encoded *e);

/* The same container bytes as dtans_encode (byte-identical to the reference
 * encode_matrix, container.py:126-204), with the per-symbol passes on CUDA
 * device `device`: validation + delta/value extraction (sparse.py:76-91,
 * 289-309), the distributions (container.py:112-114) by device radix sort +
 * run-length encode, the base pass and the backward digit pass + warp
 * interleave (codec.py:278-368, container.py:254-317), one warp per slice.
 * quantize/build_tables (entropy.py:223-436) run on the host (the one
 * floating-point step).  Host CSR in, host container out; nnz < 2^31. */
int dtans_encode_device(const dtans_csr_view *m, const dtans_encode_opts *opts, int device,
                        dtans_encoded *out);

/* Replaces quantize (entropy.py:223-321) for one domain.  symbols ascending,
 * counts >= 1.  Writes mult[n] (0 = escaped), *esc_mult, *esc_slots.
 * never_retain: n_never symbols that are always escaped. */
int dtans_quantize(int64_t n, const uint64_t *symbols, const int64_t *counts,
                   int32_t k, int32_t m, int32_t raw_width_bits,
                   int64_t n_never, const uint64_t *never_retain,
                   int32_t *mult, int32_t *esc_mult, int32_t *esc_slots);

/* ------------------------------------------------------------------ */
/* Device container (sm_100a).
 *
 * Threading (cf. spmv's `threads`, container.py:583-595): a handle is
 * immutable after upload and its launches are ordered on the stream they are
 * issued to.  Several streams may use one handle concurrently when the
 * container has no long slices and no dynamic schedule (dtans_info: the
 * plan); otherwise the per-handle scratch (partial sums of the long-slice
 * tasks, the dynamic work counter) and the host-buffer path's staging are
 * shared, so use one handle per stream or order the streams. */

typedef struct dtans_dev dtans_dev; /* opaque */

/* A container in host memory, fields as in CsrDtansContainer
 * (container.py:57-70) with the tables as the serialized record block. */
typedef struct {
    int64_t rows, cols, nnz, nslices, nwords;
    int32_t precision;
    const uint8_t *tables;       /* K * (16 | 12) bytes */
    const uint32_t *row_symbols; /* rows */
    const uint64_t *directory;   /* nslices + 1 */
    const uint32_t *stream;      /* nwords */
} dtans_container_view;

/* Upload + re-layout for the kernel (replaces the reference's in-memory
 * container + its lazily built decode arrays, container.py:344-367): the
 * shared-memory table image, and the chunk blobs (slice metadata,
 * row_symbols, stream words per chunk of slices) streamed to the device
 * through two pinned staging buffers while worker threads assemble the next
 * batch straight from the view's arrays -- which may point into an mmapped
 * CDTA file (container.py:647-720, paper_2603_01915_b200.load).  No full
 * host copy of the container is made.  Synchronous on return. */
int dtans_upload(const dtans_container_view *c, int device, dtans_dev **out);
void dtans_free(dtans_dev *h);

/* Device-memory footprint of the handle, and the launch plan it chose. */
int dtans_info(const dtans_dev *h, int64_t *device_bytes, int32_t *ctas,
               int32_t *warps_per_cta, int32_t *smem_bytes);

/* y' = A x + y on device pointers (x: cols, y/out: rows, container
 * precision).  y may be NULL (y' = A x: the power-iteration form).
 * out may alias y.  Replaces spmv (container.py:554-596) body:
 * _decode_slice_range (:370-521) fused with _accumulate_rows (:534-551).
 * Asynchronous on `stream`; errors in the stream surface in dtans_check. */
int dtans_spmv_f64(dtans_dev *h, const double *x, const double *y, double *out,
                   void *stream);
int dtans_spmv_f32(dtans_dev *h, const float *x, const float *y, float *out,
                   void *stream);

/* One power-iteration step fused into the SpMV epilogue (configs[4]; the
 * reference has no such entry: it replaces the loop body
 *   y = spmv(c, x, 0); n = ||y||; x = y / n
 * of a caller iterating the reference spmv, container.py:554-596):
 *   out = (A x) / sqrt(*sumsq_in)         (no scaling if sumsq_in is NULL)
 *   *sumsq_out += sum(out^2)              (f64 accumulation, atomic per warp)
 *   *sumsq_zero = 0                       (the next step's accumulator)
 * Device pointers; x and out in the container precision; the three scalars
 * must be distinct.  Long slices (checkpointed tasks) are scaled and summed
 * in the task / finalize kernels, so any container is accepted. */
int dtans_spmv_scaled(dtans_dev *h, const void *x, void *out, const double *sumsq_in,
                      double *sumsq_out, double *sumsq_zero, void *stream);

/* ------------------------------------------------------------------ */
/* Multi-GPU (NCCL over NVLink/NVSwitch; one process per GPU).  NCCL is
 * loaded at run time (libnccl.so.2); without it these return
 * DTANS_E_NODEVICE.  No reference counterpart: the reference is one CPU
 * process; this is the SURVEY §8b/§8e power-iteration driver. */
typedef struct dtans_mg dtans_mg; /* opaque: one NCCL communicator */

/* ncclGetUniqueId into id[128] (rank 0; share the bytes with every rank). */
int dtans_mg_unique_id(uint8_t *id);
/* ncclCommInitRank on CUDA device `device`. */
int dtans_mg_init(const uint8_t *id, int nranks, int rank, int device, dtans_mg **out);
void dtans_mg_free(dtans_mg *g);

/* Power iteration x <- A x / ||A x||_2 over row shards: this rank's handle
 * h holds rows [row_off[rank], row_off[rank+1]) of a square n x n matrix,
 * n = row_off[nranks] (distributed.shard).  x (device, n values, container
 * precision) holds x0 on entry, the same on every rank, and x_iters on exit;
 * *lambda_out = ||A x_{iters-1}||.  Per iteration: the fused scaled SpMV,
 * ncclAllReduce of sum(y^2) (one f64) and grouped ncclBroadcasts of every
 * shard's y into its row offset of the next x, all on `stream`. */
int dtans_mg_power_iteration(dtans_mg *g, dtans_dev *h, const int64_t *row_off, void *x, int iters,
                             double *lambda_out, void *stream);

/* Same product with HOST x, y, out (replaces spmv, container.py:554-596, for
 * a ctypes binding of spmv(c, x, y)): H2D copy, kernel, D2H copy,
 * synchronize, consumption check.  Pinned buffers are pipelined over slice
 * ranges on three streams (H2D / kernel / D2H); pageable buffers (numpy) are
 * staged through the handle's two pinned buffers by a pool of worker
 * threads, overlapping the host copies with the DMA. */
int dtans_spmv_host(dtans_dev *h, const void *x, const void *y, void *out);

/* Bit-exact decode on device: row_start (device, rows+1, int64) must be
 * the prefix sum of row_symbols/2; writes cols (int64) and value bit
 * patterns (u64 for f64, u32 for f32).  Replaces decode_matrix
 * (container.py:524-531). */
int dtans_decode(dtans_dev *h, const int64_t *row_start, int64_t *cols,
                 void *valbits, void *stream);

/* Synchronize `stream` and read + clear the device error word set by the
 * kernels (consumption mismatch / out-of-range column) -> DTANS_E_CORRUPT. */
int dtans_check(dtans_dev *h, void *stream);

/* Optional output row map for a row-reordered container (the encoding of
 * P*A produced by sort_rows_by_length): encoded row i is original row
 * host_map[i], so y is read and y' written at host_map[i] inside the fused
 * kernel.  host_map must be a permutation of [0, rows); NULL clears it.  An
 * extension; the container bytes stay the reference's
 * encoding of P*A. */
int dtans_set_row_map(dtans_dev *h, const uint32_t *host_map);

/* Optional column map for a symmetrically reordered container (P*A*P^T from
 * sort_symmetric_by_degree): every SpMV first gathers x'[j] = x[host_map[j]]
 * on the device (one coalesced pass over x) and multiplies with x'.  Combine
 * with dtans_set_row_map(h, same map) for y = A x in the original order.
 * host_map must be a permutation of [0, cols); NULL clears it. */
int dtans_set_col_map(dtans_dev *h, const uint32_t *host_map);

/* Number of dtANS kernels launched by this handle so far (bench evidence). */
int64_t dtans_launch_count(const dtans_dev *h);

/* The work plan dtans_upload chose (no reference counterpart: tests use it
 * to prove which kernel path a parity case ran, bench.py prints it). */
typedef struct {
    int64_t nchunks;          /* chunks of the main kernel */
    int64_t chunk_slices_max; /* most slices in one chunk */
    int64_t staged_slices;    /* slices the main kernel decodes (the rest are long) */
    int64_t nlong, ntasks, nsolo; /* long slices and their checkpointed tasks */
    int32_t dynamic;          /* atomic-ticket chunk claiming */
    int32_t dinline;          /* delta symbols inline in the slot table */
    int32_t bufb, nring;      /* staging buffer bytes, buffers per warp */
    int64_t upload_bytes;     /* bytes streamed through the pinned upload buffers */
    int64_t upload_batches;   /* cudaMemcpyAsync batches of the upload */
    int64_t pend;             /* 1: the main kernel defers the last full segment's products past a
                                 one-pair final segment's gathers (chosen per matrix) */
    int64_t nempty;           /* all-empty slices written by the empty-slice kernel (plans with
                                 long slices), outside the main kernel's chunks */
} dtans_plan_t;
int dtans_plan(const dtans_dev *h, dtans_plan_t *out);

/* Slices whose rows are summed from several task partials (long slices cut
 * into segment ranges): their y' matches the reference within the
 * north-star tolerance, every other row bitwise.  Writes up to cap slice
 * indices (ascending) to out (may be NULL); returns how many there are. */
int64_t dtans_split_slices(const dtans_dev *h, uint32_t *out, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif /* DTANS_H */
