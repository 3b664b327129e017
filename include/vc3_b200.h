/*
 * vc3_b200.h — C ABI of the B200 (sm_100a) inline 3-vector codec.
 *
 * Drop-in boundary for the hot path of the reference package `vc3`
 * (/root/reference/pkg/src/vc3).  The reference's Python layer binds numba
 * kernels (_kernels.py) through codec.py / bench.py; each entry point below
 * replaces one of those bindings (cited per function).  Differences by design:
 *   - vectors are array-of-structs float32 [n][3] (the reference splits them
 *     into three contiguous columns first, codec.py:70-83; we read the caller's
 *     (n, 3) array directly and skip those passes);
 *   - a layout travels by value (vc3_layout) and a policy as a bit mask;
 *   - every call is asynchronous on the caller's CUDA stream (`stream` is a
 *     cudaStream_t passed as void*; NULL = legacy default stream);
 *   - all pointers are DEVICE pointers unless the name ends in _host;
 *   - callers own every input and output buffer.  Per call the library
 *     allocates nothing except: vc3_error_stats (stream-ordered scratch from
 *     the device pool; vc3_error_stats_ws takes a caller workspace instead)
 *     and the host-buffer entry points (chunk staging from a library pool
 *     that keeps its memory between calls).  Once per (device, layout) the
 *     decode tables are built (vc3_prepare_layout).
 *
 * Return value: VC3_OK (0) or a negative vc3_status.  Validation happens before
 * any launch (the reference validates before its kernels, codec.py:70-83,
 * bench.py:34,47, layout.py:47-69).  Non-finite input cannot be detected before
 * the kernel on a device: compress counts offending vectors into the
 * caller-provided device counter `d_nonfinite` (may be NULL) and the host shim
 * raises NonFiniteInput after the stream sync (errors.py:12).
 */
#ifndef VC3_B200_H
#define VC3_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* BitLayout (layout.py:38-45): widths s,e,m,p,t (sum 64) and exponent bias. */
typedef struct vc3_layout {
    int32_t sign_bits;
    int32_t exponent_bits;
    int32_t mantissa_bits;
    int32_t phi_bits;
    int32_t theta_bits;
    int32_t exponent_bias;
} vc3_layout;

/* PrecisionPolicy (layout.py:119-155) as bits; a clear bit means double. */
#define VC3_THETA_SINGLE 1u
#define VC3_PHI_SINGLE 2u
#define VC3_QUANT_SINGLE 4u
#define VC3_POLICY_DEFAULT (VC3_THETA_SINGLE | VC3_QUANT_SINGLE)                   /* layout.py:183 */
#define VC3_POLICY_ORACLE 0u                                                       /* layout.py:184 */
#define VC3_POLICY_ALL_SINGLE (VC3_THETA_SINGLE | VC3_PHI_SINGLE | VC3_QUANT_SINGLE) /* layout.py:185 */

/* Numerics mode of the decoding operations (the *_ex entry points).
 *   VC3_EXACT    bit-identical to the reference: decoded components equal the
 *                reference's decode of the same word, output words equal the
 *                reference's (the plain entry points always use this mode);
 *   VC3_CONTRACT the tolerance of the north-star contract (BASELINE.json): the
 *                table decode without its exactness test, so a decoded
 *                component may be one float32 ulp from the reference's and a
 *                re-compressed word may then move by one bin at a tie.  The
 *                compress half stays bit-exact for its inputs. */
#define VC3_EXACT 0u
#define VC3_CONTRACT 1u
#define VC3_FLAGS_ALL 1u

typedef enum vc3_status {
    VC3_OK = 0,
    VC3_ERR_LAYOUT = -1,    /* BadLayout (layout.py:47-69)                  */
    VC3_ERR_ARG = -2,       /* bad pointer / negative length / bad policy   */
    VC3_ERR_CUDA = -3,      /* launch or runtime failure (vc3_last_cuda_error) */
    VC3_ERR_NONFINITE = -4, /* NonFiniteInput (host-synchronous entry points) */
    VC3_ERR_LENGTH = -5     /* LengthMismatch (bench.py:34,47)              */
} vc3_status;

/* Version / diagnostics */
const char* vc3_version(void);
const char* vc3_status_string(int status);
int vc3_last_cuda_error(void);
/* layout.py:47-69 validation, without raising */
int vc3_validate_layout(vc3_layout layout);

/* ---- the hot path -------------------------------------------------------- */

/* codec.compress (codec.py:189-202) -> _kernels.compress_kernel (_kernels.py:215-220).
 * xyz: float32 [n][3]; words: uint64 [n]. */
int vc3_compress(const float* xyz, uint64_t* words, int64_t n, vc3_layout layout,
                 uint32_t policy, int32_t* d_nonfinite, void* stream);

/* The bound, relative to the magnitude, by which the fast table decode's
 * components can differ from the reference's doubles (measured on the host
 * over every table index against the reference's tables when the tables are
 * built); components within it of a float32 rounding boundary are
 * re-evaluated exactly.  0 for layouts decoded without tables.  Builds the
 * tables on first use. */
int vc3_decode_tolerance(vc3_layout layout, double* tol);

/* Build the decode tables of a layout on the current device ahead of the
 * first operation (the 49 KB fast table, and for VC3_EXACT the reference's
 * 6 MB tables).  Optional: every operation builds them on first use, also
 * inside a caller's CUDA-graph capture (the build uses a private stream and
 * relaxed capture mode), but preparing keeps that one-off host work (~10 ms)
 * out of the first call. */
int vc3_prepare_layout(vc3_layout layout, uint32_t flags);

/* codec.decompress (codec.py:205-228) -> decompress_kernel_tab/_direct
 * (_kernels.py:293-331).  words: uint64 [n]; xyz: float32 [n][3].
 * Bit-identical to the reference's decode (its libm sin/cos tables): the
 * first call for a layout builds a 49 KB shared-memory table and the 6 MB
 * reference table on the device (capture-safe; see vc3_prepare_layout). */
int vc3_decompress(const uint64_t* words, float* xyz, int64_t n, vc3_layout layout,
                   void* stream);
/* vc3_decompress with a numerics mode (VC3_EXACT / VC3_CONTRACT). */
int vc3_decompress_ex(const uint64_t* words, float* xyz, int64_t n, vc3_layout layout,
                      uint32_t flags, void* stream);

/* vc3_compress and the magnitude events of the same vectors in one pass
 * (codec.py:241-262): d_events[0] += flushed, d_events[1] +=
 * saturated (device uint64[2], zeroed by the caller). */
int vc3_compress_events(const float* xyz, uint64_t* words, int64_t n, vc3_layout layout,
                        uint32_t policy, int32_t* d_nonfinite, uint64_t* d_events, void* stream);

/* bench.add_compressed (bench.py:41-69) -> add_compressed_kernel (_kernels.py:348-359):
 * c = compress(decompress(a) + decompress(b)) fused, nothing uncompressed
 * touches memory.  The reference's default policy here is ALL_SINGLE. */
int vc3_add_compressed(const uint64_t* a, const uint64_t* b, uint64_t* c, int64_t n,
                       vc3_layout layout, uint32_t policy, void* stream);
/* vc3_add_compressed with a numerics mode (VC3_EXACT / VC3_CONTRACT). */
int vc3_add_compressed_ex(const uint64_t* a, const uint64_t* b, uint64_t* c, int64_t n,
                          vc3_layout layout, uint32_t policy, uint32_t flags, void* stream);

/* bench.add_raw (bench.py:30-38) -> add_raw_kernel (_kernels.py:341-345):
 * the uncompressed float32 baseline, c[i] = a[i] + b[i] over n_floats floats. */
int vc3_add_raw(const float* a, const float* b, float* c, int64_t n_floats, void* stream);

/* No reference symbol: y_out = compress(alpha*decompress(x) + decompress(y)).
 * float32 ops: t = alpha*x (rounded), then t + y (rounded), per component.
 * y_out may alias y (in-place update). */
int vc3_axpy(float alpha, const uint64_t* x, const uint64_t* y, uint64_t* y_out, int64_t n,
             vc3_layout layout, uint32_t policy, void* stream);
int vc3_axpy_ex(float alpha, const uint64_t* x, const uint64_t* y, uint64_t* y_out, int64_t n,
                vc3_layout layout, uint32_t policy, uint32_t flags, void* stream);

/* Low-storage (2N) RK stage on compressed registers (SURVEY §8a R18,
 * PAPER.md:135,336), all three operands stored compressed:
 *   dq' = a*dq + dt*R ;  q' = q + b*dq'
 * float32 per component, each product and sum rounded in that order; q' uses
 * the register value of dq' (before it is re-compressed).  q and dq are
 * updated in place (40 B of HBM traffic per vector). */
int vc3_rk_stage(float a, float b, float dt, uint64_t* q, uint64_t* dq, const uint64_t* R,
                 int64_t n, vc3_layout layout, uint32_t policy, void* stream);
int vc3_rk_stage_ex(float a, float b, float dt, uint64_t* q, uint64_t* dq, const uint64_t* R,
                    int64_t n, vc3_layout layout, uint32_t policy, uint32_t flags, void* stream);

/* Uncompressed float32 baseline of vc3_rk_stage (60 B of HBM traffic per
 * vector): the same op order on flat float32 arrays of n_floats elements. */
int vc3_rk_stage_f32(float a, float b, float dt, float* q, float* dq, const float* R,
                     int64_t n_floats, void* stream);

/* ---- pieces (codec.py:99-186) -------------------------------------------- */

/* codec.to_spherical (codec.py:99-114) -> spherical_kernel (_kernels.py:223-229) */
int vc3_to_spherical(const float* xyz, double* r, double* theta, double* phi, int64_t n,
                     uint32_t policy, int32_t* d_nonfinite, void* stream);
/* codec.quantize_angles (codec.py:122-140) -> quantize_kernel (_kernels.py:232-237) */
int vc3_quantize_angles(const double* theta, const double* phi, int64_t* n_theta,
                        int64_t* n_phi, int64_t n, vc3_layout layout, uint32_t policy,
                        void* stream);
/* codec.dequantize_angles (codec.py:143-153) -> dequantize_kernel (_kernels.py:334-338) */
int vc3_dequantize_angles(const int64_t* n_theta, const int64_t* n_phi, double* theta,
                          double* phi, int64_t n, vc3_layout layout, void* stream);
/* codec.encode_magnitude (codec.py:156-175) -> encode_mag_kernel (_kernels.py:240-243) */
int vc3_encode_magnitude(const double* r, uint64_t* field, int64_t n, vc3_layout layout,
                         void* stream);
/* codec.decode_magnitude (codec.py:178-186) -> decode_mag_kernel (_kernels.py:246-249) */
int vc3_decode_magnitude(const int64_t* field, float* r, int64_t n, vc3_layout layout,
                         void* stream);
/* codec.magnitude_event_counts (codec.py:241-262): d_counts[0] += flushed,
 * d_counts[1] += saturated (caller zeroes them). */
int vc3_magnitude_events(const float* xyz, int64_t n, vc3_layout layout,
                         unsigned long long* d_counts, void* stream);
/* The same, also counting vectors with a NaN or infinite component into
 * *d_nonfinite (device int32, zeroed by the caller; the reference raises
 * NonFiniteInput for them, codec.py:76-78). */
int vc3_magnitude_events_checked(const float* xyz, int64_t n, vc3_layout layout,
                                 unsigned long long* d_counts, int32_t* d_nonfinite, void* stream);

/* ---- K7 variants (analysis.py:259-417) ------------------------------------
 * Angle coding variants the reference evaluates in compand_study and
 * split_sweep, as word formats (ours: the reference defines none):
 *   compander: the layout's packing [magnitude | n_phi | n_theta] with
 *              companded indices (Compander.encode/decode, analysis.py:342-393);
 *   split:     [magnitude | J], J = n_phi*(n_theta_max+1) + n_theta in
 *              total_bits = phi_bits + theta_bits (SplitConfig, joint_encode,
 *              analysis.py:259-297).
 * Angles use the reference's double pipeline (ORACLE policy); the decode
 * uses double sin/cos and narrows to float32 like compand_study/split_sweep. */
#define VC3_VARIANT_UNIFORM 0
#define VC3_VARIANT_COSINE 1
#define VC3_VARIANT_TANH 2
#define VC3_VARIANT_SPLIT 3

typedef struct vc3_variant {
    int32_t kind;       /* VC3_VARIANT_* */
    int32_t total_bits; /* split: joint index width (must equal phi_bits + theta_bits) */
    int64_t n_phi_max;  /* split: n_phi_max (n_theta_max is derived, analysis.py:271-276) */
    double gamma;       /* tanh compander strength (> 0) */
} vc3_variant;

int vc3_compress_variant(const float* xyz, uint64_t* words, int64_t n, vc3_layout layout,
                         vc3_variant variant, int32_t* d_nonfinite, void* stream);
int vc3_decompress_variant(const uint64_t* words, float* xyz, int64_t n, vc3_layout layout,
                           vc3_variant variant, void* stream);
/* bucket maxima the variant uses (split: derived n_theta_max) */
int vc3_variant_maxima(vc3_layout layout, vc3_variant variant, int64_t* n_theta_max,
                       int64_t* n_phi_max);

/* ---- statistics (analysis.py:118-167) ------------------------------------ */

/* Per-chunk error moments, in double: for chunk k (chunk vectors each, last
 * one ragged) writes d_chunk_stats[4k..4k+3] = (count, mean, M2, max).
 * Chunks merge on the host (or across ranks) in chunk order exactly like
 * analysis._Welford.  kind selects the per-vector error e_i:
 *   VC3_ERR_L2             ||v - vh||_2                 (analysis.py:148-154)
 *   VC3_ERR_L2_NORMALISED  ||v - vh||_2 / ||v||_2        (normalised=True)
 *   VC3_ERR_ANGULAR        atan2(||v x vh||, v . vh), radians
 *   VC3_ERR_REL_MAGNITUDE  | ||vh|| - ||v|| | / ||v||
 * The last two are not in the reference; their op order
 * is fixed and restated on the CPU by the test suite.  0/1 keep the meaning of
 * the reference's `normalised` flag. */
#define VC3_ERR_L2 0
#define VC3_ERR_L2_NORMALISED 1
#define VC3_ERR_ANGULAR 2
#define VC3_ERR_REL_MAGNITUDE 3
int vc3_error_stats(const float* v, const float* vh, int64_t n, int32_t kind,
                    int64_t chunk, double* d_chunk_stats, void* stream);
/* The same with a caller-provided device workspace of at least
 * vc3_error_stats_workspace(n, chunk) bytes (no allocation at all). */
int vc3_error_stats_workspace(int64_t n, int64_t chunk, uint64_t* bytes);
int vc3_error_stats_ws(const float* v, const float* vh, int64_t n, int32_t kind, int64_t chunk,
                       double* d_chunk_stats, void* d_work, uint64_t work_bytes, void* stream);

/* ---- flux-reconstruction flux divergence (Alg. 1) ------
 * No reference code exists; the operation is the paper's
 * Algorithm 1 for step 10 of its FR table:
 *   div[(k*n_vars + c)*ld + i] = sum_j sum_d D[(d*n_points + j)*n_points + k]
 *                                * X_d(words[(j*n_vars + c)*ld + i])
 * with X = decompress(word) (vc3_decompress), D the 3*n_points x n_points
 * divergence operator (float32, row-major, device memory), i < n_elem the
 * element, c < n_vars the equation, n_points <= 256 solution points per
 * element and ld >= n_elem the element stride.  Runs on the tcgen05 tensor
 * cores with fp32-accurate operand splitting (3xTF32).
 *
 * vc3_fr_prepare_operator splits D into the kernel's staged operator
 * (vc3_fr_operator_floats(n_points) floats of device memory, 16-B aligned);
 * prepare once per operator, reuse for every call. */
int64_t vc3_fr_operator_floats(int n_points);
int vc3_fr_prepare_operator(const float* D, int n_points, float* op, void* stream);
int vc3_fr_divergence(const uint64_t* words, const float* op, float* div, int64_t n_elem,
                      int n_vars, int64_t ld, int n_points, vc3_layout layout, void* stream);
/* Uncompressed baseline: flux[((j*n_vars + c)*ld + i)*3 + d] float32. */
int vc3_fr_divergence_f32(const float* flux, const float* op, float* div, int64_t n_elem,
                          int n_vars, int64_t ld, int n_points, void* stream);

/* Tensor-product hexahedra of degree 1..4 (n_points = (degree+1)^3, point
 * index px + n py + n^2 pz): the same divergence with D built from the 1D
 * derivative matrix m1d[a*(degree+1) + m] = l_m'(x_a) (HOST memory, read at
 * launch), sum-factorised on the CUDA cores (3(degree+1) multiply-adds per
 * output).  Table layouts only (angle fields <= 20 bits). */
int vc3_fr_divergence_hex(const uint64_t* words, const float* m1d, int degree, float* div,
                          int64_t n_elem, int n_vars, int64_t ld, vc3_layout layout, void* stream);
int vc3_fr_divergence_hex_f32(const float* flux, const float* m1d, int degree, float* div,
                              int64_t n_elem, int n_vars, int64_t ld, void* stream);

/* ---- host-buffer entry points (reference-facing, synchronous) ------------
 * Same operations on HOST arrays: the call streams chunks host->device, runs
 * the kernel and copies results back, overlapping copies and compute on
 * internal streams.  Pinned host memory gives full PCIe/C2C bandwidth;
 * pageable memory works but is slower.  Returns after the results are in
 * the host buffer.  device: CUDA ordinal to run on. */
int vc3_add_compressed_host(const uint64_t* a_host, const uint64_t* b_host, uint64_t* c_host,
                            int64_t n, vc3_layout layout, uint32_t policy, int32_t device);
int vc3_compress_host(const float* xyz_host, uint64_t* words_host, int64_t n, vc3_layout layout,
                      uint32_t policy, int64_t* nonfinite_out, int32_t device);
int vc3_decompress_host(const uint64_t* words_host, float* xyz_host, int64_t n,
                        vc3_layout layout, int32_t device);

#ifdef __cplusplus
}
#endif
#endif /* VC3_B200_H */
