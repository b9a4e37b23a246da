/*
 * isf_lossy.h -- C ABI of the B200-native in-situ lossy compressor.
 *
 * This is the drop-in boundary for the one hot path of arXiv 2407.20731's
 * in-situ framework (SPEC.md MODULE tasks): error-bounded lossy compression of
 * spectral-element fp64 fields by a per-element 3-D discrete Legendre transform
 * (north_star; SPEC.md:205 names a DCT), energy
 * truncation and mask + packed-value encoding, decompression and error report.
 *
 * The reference declares, but never implements, this interface:
 *   - proj/include/isf/core/frame.hpp:11   "payload_kind 1 carries a compressed
 *                                           block (see tasks/lossy.hpp)"  -- absent
 *   - SPEC.md:222  lossy_compress(f: Field, cfg: LossyConfig) -> CompressedBlock
 *   - SPEC.md:231  lossy_decompress(b: CompressedBlock, shape) -> Field
 *   - SPEC.md:212-215  CompressionReport / Eq. 1
 *   - proj/include/isf/core/errors.hpp:8-38  ErrorCode (status codes below)
 * include/isf/tasks/lossy.hpp is the C++ host API (the missing tasks/lossy.hpp)
 * written on top of these entry points; INTEGRATION.md shows the binding.
 *
 * Conventions
 *   - Every entry point returns 0 on success, otherwise 1 + (int)isf::ErrorCode
 *     (ISF_E_* below).  No C++ exception crosses the ABI.  The message of the last
 *     failure on the calling thread is isf_lossy_last_error().
 *   - Device pointers are plain CUDA device pointers owned by the caller; the
 *     field must be 16-byte aligned.  `cuda_stream` is a cudaStream_t (NULL =
 *     legacy default stream).  *_async calls only enqueue work on that stream.
 *   - Handoff rule (proj/include/isf/staging/staging.hpp:5-9): the
 *     field must not be overwritten until compress has completed on the stream.
 *   - One plan per (device, points-per-axis, components) and per stream at a time
 *     (single-owner, like StageWriter).
 *
 * Stream format (little-endian, proj/include/isf/core/bytes.hpp:17-32):
 *   counts u32[B] | zero pad to 16 B | masks u64[B][W] | values f64[sum counts]
 *   B = elements * components blocks, block b = element*components + component,
 *   W = ceil(P^3/64), mask bit j (LSB first) <-> Legendre coefficient j =
 *   kx + P*(ky + P*kz); values in ascending j, blocks in order.
 */
#ifndef ISF_LOSSY_H
#define ISF_LOSSY_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* 1 + isf::ErrorCode (proj/include/isf/core/errors.hpp:8-38) */
enum {
    ISF_OK = 0,
    ISF_E_LENGTH_MISMATCH = 1 + 2,      /* ErrorCode::LengthMismatch      */
    ISF_E_SERIALIZATION_FAILED = 1 + 4, /* ErrorCode::SerializationFailed */
    ISF_E_SHAPE_MISMATCH = 1 + 12,      /* ErrorCode::ShapeMismatch       */
    ISF_E_UNKNOWN_CODEC = 1 + 13,       /* ErrorCode::UnknownCodec        */
    ISF_E_TASK_FAILED = 1 + 17,         /* ErrorCode::TaskFailed (CUDA / NCCL failure) */
    ISF_E_INVALID_ARGUMENT = 1 + 20     /* ErrorCode::InvalidArgument     */
};

/* LossyConfig.error_norm.  RelativeL2: exact Parseval energy rule
 * (DESIGN.md 3.4), in the GLL-quadrature norm ||v||_w^2 = sum w_x w_y w_z v^2, i.e. the
 * L2 norm of the element polynomials (the norm of NEKO's DLT; err2 / nrm2 below report
 * it).  It bounds the plain point-sample relative L2 only up to sqrt(max w / min w) per
 * element (about 40 at lx = 8; tests/test_oracle_norms.py), which is why SPEC.md's
 * DCT-II wording (plain samples) and this transform differ.  RelativeLInf: per block, sum over the discarded coefficients of
 * |a_j| * max|basis_j| <= max_error * max|u| (a bound on the reconstruction's max
 * error; runs on the generic kernels). */
enum { ISF_NORM_RELATIVE_L2 = 0, ISF_NORM_RELATIVE_LINF = 1 };

/* status bits in isf_lossy_stats.status */
enum { ISF_STATUS_NONFINITE = 1, ISF_STATUS_SHAPE = 2, ISF_STATUS_OVERFLOW = 4 };

/* Per-call scalars.  Compress fills kept/blocks/stream_bytes/field_bytes and the
 * coefficient-space energies (Parseval estimate of the L2 error); decompress with
 * an original fills the measured GLL-weighted L2 and Linf terms.  Layout is
 * fixed (12 x 8 bytes) so that it can be all-reduced as two arrays. */
typedef struct isf_lossy_stats {
    double err2;           /* sum_w (u - u~)^2                                   */
    double nrm2;           /* sum_w u^2                                          */
    double err_inf;        /* max |u - u~|                                       */
    double u_inf;          /* max |u|                                            */
    double disc2;          /* coefficient energy of the discarded set (upper bound) */
    double tot2;           /* coefficient energy of the block (lower bound)        */
    uint64_t kept;         /* retained coefficients                              */
    uint64_t blocks;       /* (element, component) blocks                        */
    uint64_t stream_bytes; /* encoded stream bytes (CompressionReport.compressed_size) */
    uint64_t field_bytes;  /* raw field bytes (CompressionReport.original_size)  */
    uint64_t status;       /* ISF_STATUS_* bits                                  */
    uint64_t reserved;
} isf_lossy_stats;

typedef struct isf_lossy_plan isf_lossy_plan;

/* Plan: owns the constant GLL operators on `device`, the decoupled look-back
 * tile descriptors and reduction workspace.  P in [2,16], components in {1,3}
 * (proj/src/core/types.cpp:59-64). */
int isf_lossy_plan_create(isf_lossy_plan** plan, uint32_t points_per_element_axis,
                          uint32_t components, int device);
int isf_lossy_plan_destroy(isf_lossy_plan* plan);

/* Upper bound of the stream size for n_elements elements (incompressible data). */
uint64_t isf_lossy_stream_capacity(uint32_t points_per_element_axis, uint32_t components,
                                   uint64_t n_elements);
/* Bytes of the counts + masks prefix of the stream. */
uint64_t isf_lossy_stream_header_bytes(uint32_t points_per_element_axis, uint32_t components,
                                       uint64_t n_elements);

/* Compress a device-resident field.  Enqueues the kernels and
 * writes an isf_lossy_stats to DEVICE memory d_stats (nothing is copied back). */
int isf_lossy_compress_async(isf_lossy_plan* plan, const double* d_field, uint64_t n_elements,
                             double max_error, int error_norm, void* d_stream, uint64_t capacity,
                             isf_lossy_stats* d_stats, void* cuda_stream);
/* Same, then synchronises and returns the stream size / stats on the host; maps
 * non-finite input to ISF_E_INVALID_ARGUMENT (proj/src/core/types.cpp:71-73) and
 * a too-small capacity to ISF_E_SERIALIZATION_FAILED. */
int isf_lossy_compress(isf_lossy_plan* plan, const double* d_field, uint64_t n_elements,
                       double max_error, int error_norm, void* d_stream, uint64_t capacity,
                       uint64_t* stream_bytes, isf_lossy_stats* stats, void* cuda_stream);

/* Decompress.  If d_original is not NULL the GLL-weighted L2
 * and Linf error terms against it are accumulated.  An inconsistent stream (count
 * != popcount(mask), bits beyond P^3, size mismatch) is ISF_E_SHAPE_MISMATCH. */
int isf_lossy_decompress_async(isf_lossy_plan* plan, const void* d_stream, uint64_t stream_bytes,
                               uint64_t n_elements, double* d_out, const double* d_original,
                               isf_lossy_stats* d_stats, void* cuda_stream);
int isf_lossy_decompress(isf_lossy_plan* plan, const void* d_stream, uint64_t stream_bytes,
                         uint64_t n_elements, double* d_out, const double* d_original,
                         isf_lossy_stats* stats, void* cuda_stream);

/* Host-buffer entry points (what a CPU-side caller of the reference API binds):
 * H2D of the field, compress, D2H of the stream, all inside the call.  Host
 * buffers may be pageable; pinned buffers are faster. */
int isf_lossy_compress_host(isf_lossy_plan* plan, const double* h_field, uint64_t n_elements,
                            double max_error, int error_norm, void* h_stream, uint64_t capacity,
                            uint64_t* stream_bytes, isf_lossy_stats* stats);
int isf_lossy_decompress_host(isf_lossy_plan* plan, const void* h_stream, uint64_t stream_bytes,
                              uint64_t n_elements, double* h_out, const double* h_original,
                              isf_lossy_stats* stats);

/* Global reduction of per-rank stats over an NCCL communicator (ncclComm_t):
 * sum of err2,nrm2,disc2,tot2 (f64) and kept,blocks,stream_bytes,field_bytes
 * (u64), max of err_inf,u_inf (f64), bitwise-or folded into status via max.
 * NCCL is resolved at run time from the process (dlsym), so the library has no
 * link-time NCCL dependency and uses whichever NCCL created the communicator. */
int isf_lossy_allreduce(isf_lossy_stats* d_stats, void* nccl_comm, void* cuda_stream);
/* The same over n consecutive records d_stats[0..n) (1 <= n <= 256, e.g. the four
 * fields of a step) in one NCCL group: three all-reduces whatever n is.  The NCCL
 * symbols come from the libnccl instance already loaded in the process (the one that
 * created the communicator), else from the global scope. */
int isf_lossy_allreduce_n(isf_lossy_stats* d_stats, uint32_t n, void* nccl_comm, void* cuda_stream);

/* Device CRC-32 (IEEE / zlib polynomial; replaces the host zlib call of
 * proj/src/core/crc32.cpp:7-20 for device-resident data): *d_crc = crc32(d_data[0..n)).
 * Asynchronous on cuda_stream; any alignment (16-byte aligned data takes the fast path). */
int isf_lossy_crc32(isf_lossy_plan* plan, const void* d_data, uint64_t n, uint32_t* d_crc,
                    void* cuda_stream);

/* Kind-1 frame on the device (proj/include/isf/core/frame.hpp:3-11,
 * proj/src/core/frame.cpp:9-25 build_frame) with SPEC.md:282's payload, converted on
 * the device from the compressed stream d_stream (n_elements elements; the stats of
 * that compress call in d_stats, read on the device):
 *   [0,48) header "ISF1" | 1 | kind 1 | step | sim_time | E | P | components | 0 | payload_len
 *   payload: kept_count u32[n_elements] | index u32[K] | value f64[K] |
 *            codec id u16 = 0 | coded length u64 = 0 (no lossless stage yet)
 *   CRC-32 u32 of all preceding bytes
 * K = d_stats->kept; index = component * P^3 + j (j = kx + P (ky + P kz)), ascending
 * inside each element, values in the same order.  The frame is
 * ISF_FRAME_OVERHEAD + 4 n_elements + 12 K bytes (at most isf_lossy_frame_capacity);
 * a frame_cap that is too small sets ISF_STATUS_OVERFLOW in d_stats->status.  d_frame
 * and d_stream are 16-byte aligned and distinct; fully asynchronous. */
#define ISF_FRAME_OVERHEAD 62
int isf_lossy_frame_async(isf_lossy_plan* plan, void* d_frame, uint64_t frame_cap, const void* d_stream,
                          uint64_t n_elements, const isf_lossy_stats* d_stats, uint32_t elements_per_axis,
                          uint64_t step_index, double sim_time, void* cuda_stream);
/* Worst-case kind-1 frame bytes (every coefficient kept). */
uint64_t isf_lossy_frame_capacity(uint32_t points_per_element_axis, uint32_t components, uint64_t n_elements);

/* Eq. 1: (original - compressed) / original in fp64. */
double isf_lossy_compression_ratio(uint64_t original_size, uint64_t compressed_size);

/* Diagnostics / tests. */
const char* isf_lossy_last_error(void);
const char* isf_lossy_error_code_name(int status);
int isf_lossy_plan_operators(const isf_lossy_plan* plan, double* F, double* B, double* x,
                             double* w);
/* Number of kernel launches the last compress / decompress call enqueued. */
int isf_lossy_plan_last_launches(const isf_lossy_plan* plan);
/* lx = 8 compress schedule.  ISF_COMPRESS_TWO_PASS: kept values go to per-block slots
 * and a second kernel packs them (best when few coefficients are kept, the in-situ CFD
 * case).  ISF_COMPRESS_SINGLE_PASS: the values are written to their final place by the
 * selecting kernel two rounds later, behind per-round CTA aggregates (no slot round
 * trip: best for weakly compressible data, C/F > ~0.5).  ISF_COMPRESS_AUTO (default):
 * single-pass when the plan's last completed compress kept more than half of the
 * coefficients (read from host-mapped memory the kernels write: no synchronisation).
 * Streams are byte-identical either way.  Returns the previous mode, or < 0 on error. */
#define ISF_COMPRESS_TWO_PASS 0
#define ISF_COMPRESS_SINGLE_PASS 1
#define ISF_COMPRESS_AUTO 2
int isf_lossy_plan_set_compress_mode(isf_lossy_plan* plan, int mode);
/* Device generator of the synthetic inputs: the in-situ producer
 * stand-in.  which: 0=u 1=v 2=w 3=p of the t=0 Taylor-Green vortex at GLL nodes
 * for element z-layers [ez0, ez0+nz) of an E_ax^2 x E_z mesh. */
int isf_lossy_generate_tgv(isf_lossy_plan* plan, double* d_out, uint32_t E_ax, uint32_t ez0,
                           uint32_t nz, int which, double domain, void* cuda_stream);
/* Spectral field: coefficients (2U-1)*amp[j] with U from Philox4x32-10, then the
 * inverse DLT (uses the decompress kernel on a dense stream built on device). */
int isf_lossy_generate_spectral(isf_lossy_plan* plan, double* d_out, uint64_t block0,
                                uint64_t nblocks, uint64_t seed, const double* h_amp,
                                void* cuda_stream);

/* Async in-situ mode (cfg5): a memory-bound solver stand-in step
 * dst = src + alpha*(aux - src) on `cuda_stream` (reads 2n, writes n doubles). */
int isf_lossy_solver_standin(double* d_dst, const double* d_src, const double* d_aux, uint64_t n,
                             double alpha, void* cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* ISF_LOSSY_H */
