/*
 * isf_oracle.h -- CPU ORACLE for the in-situ lossy-compression hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2407_20731_b200/,
 * include/) links, loads or calls this code.  It is used by tests/ (as the
 * checker), by __graft_entry__.smoke() (as the checker) and by bench.py's
 * cpu_baseline / --impl reference leg (as the CPU baseline: the reference
 * ships no implementation of this path).
 *
 * What it restates (citations relative to /root/reference):
 *   - SPEC.md:204-215   LossyConfig / CompressedBlock / CompressionReport (Eq. 1)
 *   - SPEC.md:222-239   lossy_compress / lossy_decompress: per element and
 *                       component, orthonormal transform -> sort |c| desc ->
 *                       smallest prefix with discarded/total energy <= eps^2
 *   - SPEC.md:268-273   error guarantee, Parseval, Eq.1 exactness, monotonicity
 *   - proj/include/isf/core/types.hpp:20-24,51-53   Field layout
 *     index = (element*P^3 + point)*components + component, point = px+P*(py+P*pz)
 *   - proj/include/isf/core/bytes.hpp:17-32          little-endian encoding
 *   - BASELINE.json north_star: the transform is the Legendre/GLL DLT (not the
 *     DCT of SPEC.md:205,275) -- definitions pinned in DESIGN.md section 3.
 *
 * PARITY STATUS: the reference has no implementation and no golden vectors for
 * this path ("parity unpinned" by reference tests).  The
 * oracle is pinned by SPEC's worked examples and
 * properties, by an independent numpy restatement
 * (tests/golden/make_golden.py) and, for the frame format, by the reference's
 * own build_frame compiled from /root/reference (oracle/_ref).
 */
#ifndef ISF_ORACLE_H
#define ISF_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same layout as isf_lossy_stats in include/isf_lossy.h (kept separate on purpose:
 * the oracle does not include product headers). */
typedef struct {
    double err2;      /* sum_w (u-u~)^2  (GLL-weighted, decompress with original) */
    double nrm2;      /* sum_w u^2                                                  */
    double err_inf;   /* max |u-u~|                                                 */
    double u_inf;     /* max |u|                                                    */
    double disc2;     /* coefficient-space discarded energy (hi-sum, upper bound, scaled) */
    double tot2;      /* coefficient-space total energy     (same quantisation)      */
    uint64_t kept;    /* total kept coefficients                                     */
    uint64_t blocks;  /* number of (element, component) blocks                       */
    uint64_t stream_bytes;
    uint64_t field_bytes;
    uint64_t status;  /* bit 0: non-finite input, bit 1: shape mismatch, bit 2: overflow */
    uint64_t reserved;
} iso_stats;

/* ---- GLL operators ---- */
int iso_gll(int lx, double* x, double* w);
int iso_matrices(int lx, double* F /* [k*lx+i] */, double* B /* [i*lx+k] */);

/* ---- one block (lx^3 contiguous values, x fastest) ---- */
void iso_fwd_block(int lx, const double* F, const double* u, double* a);   /* sweeps z, y, x */
void iso_inv_block(int lx, const double* B, const double* a, double* u);   /* sweeps x, y, z */
/* Pinned truncation rule v2.  Writes ceil(lx^3/64) mask words,
 * returns kept count; *lo_total (block total at scale A) / *lo_disc (sum hi over the
 * discarded set at scale B) receive the integer energy sums and scale_exp[0..1] the
 * binary exponents that map them back (energy = lo_total * 2^scale_exp[0],
 * lo_disc * 2^scale_exp[1]). */
uint32_t iso_select_block(int lx, const double* a, double max_error, uint64_t* mask,
                          uint64_t* lo_total, uint64_t* lo_disc, int* scale_exp, int* nonfinite);
/* Same rule with the threshold perturbed: thr' = floor(thr * (1 + rel)) (rel may be
 * negative).  Used by the parity tests' near-threshold acceptance rule. */
uint32_t iso_select_block_perturbed(int lx, const double* a, double max_error, double rel,
                                    uint64_t* mask);

/* SPEC-literal rule (SPEC.md:225 in exact reals, binary128-filtered): kept count
 * and mask; *ambiguous = 1 when binary128 cannot decide the cut (exact fallback in
 * oracle.py).  rel scales eps^2 * T by (1 + rel). */
uint32_t iso_select_block_literal(int lx, const double* a, double max_error, double rel, uint64_t* mask,
                                  int* ambiguous);
/* Whole-field comparison of a stream's masks with the literal rule; cls[b]: 0 same,
 * 1 differs within SURVEY.md 8c's near-threshold band, 2 differs beyond it,
 * 3 ambiguous.  Returns the count of cls != 0. */
uint64_t iso_literal_check(int lx, int comps, uint64_t n_elements, const double* field, double max_error,
                           const uint8_t* stream, uint8_t* cls, uint64_t* kept_literal, int nthreads);

/* RelativeLInf rule: Bm = synthesis matrix [i*lx+k], umax = max|u| of the
 * block's nodal values.  Returns the kept count and writes the mask. */
uint32_t iso_select_block_linf(int lx, const double* Bm, const double* a, double umax, double max_error,
                               uint64_t* mask, int* nonfinite);

/* ---- whole fields ---- */
uint64_t iso_stream_capacity(int lx, uint64_t nblocks);
uint64_t iso_stream_header_bytes(int lx, uint64_t nblocks);  /* counts + masks */
/* returns 0 or 1+ErrorCode (13 = ShapeMismatch, 21 = InvalidArgument) */
int iso_compress(int lx, int comps, uint64_t n_elements, const double* field, double max_error,
                 uint8_t* stream, uint64_t cap, uint64_t* stream_bytes, iso_stats* st, int nthreads);
/* norm: 0 = RelativeL2, 1 = RelativeLInf */
int iso_compress_norm(int lx, int comps, uint64_t n_elements, const double* field, double max_error, int norm,
                      uint8_t* stream, uint64_t cap, uint64_t* stream_bytes, iso_stats* st, int nthreads);
int iso_decompress(int lx, int comps, uint64_t n_elements, const uint8_t* stream,
                   uint64_t stream_bytes, double* out, const double* original, iso_stats* st,
                   int nthreads);
/* Forward transform of every block (coefficients in block order, lx^3 per block). */
void iso_forward_field(int lx, int comps, uint64_t n_elements, const double* field, double* coeffs,
                       int nthreads);

/* ---- synthetic inputs ---- */
/* TGV at t=0 sampled at GLL nodes; which: 0=u 1=v 2=w 3=p.  Elements ez in [ez0, ez0+nz)
 * of an E_ax x E_ax x E_z mesh with element edge h = domain/E_ax. */
void iso_gen_tgv(int E_ax, int lx, int which, uint32_t ez0, uint32_t nz, double domain,
                 double* out, int nthreads);
/* Spectral field: coefficient a_klm = (2U-1) * amp[k,l,m], U = 53-bit uniform from
 * Philox4x32-10(key = (seed lo32, seed hi32), counter = (block lo32, block hi32,
 * j = k+lx*(l+lx*m), 0)), U = (r0 << 21 | r1 >> 11) * 2^-53; nodal = inverse DLT. */
void iso_spectral_amplitudes(int lx, double decay_s, double* amp /* lx^3 */);
void iso_gen_spectral(int lx, uint64_t block0, uint64_t nblocks, uint64_t seed, double decay_s,
                      double* out, int nthreads);
void iso_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

#ifdef __cplusplus
}
#endif
#endif
