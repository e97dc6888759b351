/*
 * minplus.h -- C ABI of the B200 (sm_100a) hot path of arXiv 2409.17688,
 * "HPC acceleration of large (min,+) matrix products to compute domination-type
 * parameters in graphs".
 *
 * Citations: "P:L" = the paper's PAPER.md line L (section / equation / algorithm named
 * beside it); "S:L" = SPEC.md line L; "G<k>" = a reading of the paper listed in DESIGN.md.
 * Notation (G1): n = order of the path P_n (the paper's m), m = length of the cycle C_m
 * (the paper's n), N = |C_n| = number of correct n-words = order of A(D_n).
 *
 * Conventions shared by every entry point
 *   - Tropical values are uint16_t.  MP_INF = 0xFFFF is +inf; finite values are
 *     0..MP_FINITE_MAX.  s(a,b) = a+b if both are finite and a+b <= MP_FINITE_MAX, else
 *     +inf (G6; P:53 defines the semiring, P:250 fixes 16-bit storage).
 *   - Matrices are row-major; "ld" is the row pitch in elements.
 *   - No exception crosses the ABI.  Every call returns an mp_status; on a non-OK status
 *     the outputs are left untouched and mp_last_error() returns a thread-local message.
 *   - Calls serialise on a process-wide mutex.  GPU work runs on the calling thread's
 *     current CUDA device (cudaSetDevice / torch.cuda.set_device before the call).
 *   - There is no CPU fallback: if no sm_100 device is present, calls that compute
 *     return MP_ERR_CUDA.
 */
#ifndef MINPLUS_H
#define MINPLUS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MP_INF 0xFFFFu        /* +inf at the boundary                  */
#define MP_FINITE_MAX 0x7FFEu /* largest finite input; a finite sum above it is +inf (G6) */
#define MP_MAX_K 256          /* largest power index a periodic result can describe        */
#define MP_MAX_N 13           /* largest path order n: 13 is the paper's future work (P:250,
                                 P:551: 34.6 GB per matrix exceeded its 32 GB GPU)           */

typedef enum {
    MP_OK = 0,
    MP_ERR_DOMAIN = 1,       /* n < 2 or n > MP_MAX_N, cycle m < 3 (G17), dims <= 0, NULL
                                pointers, ld < cols, C aliasing A or B */
    MP_ERR_RANGE = 2,        /* an input entry in (MP_FINITE_MAX, MP_INF)                   */
    MP_ERR_RESOURCE = 3,     /* device or host memory budget exceeded; mp_last_error()
                                names the byte count                                 */
    MP_ERR_NOT_PERIODIC = 4, /* no repeat A^k = c (x) A^j with k <= max_k (G20)             */
    MP_ERR_CUDA = 5,         /* a CUDA runtime error, or no sm_100 device                   */
    MP_ERR_COMM = 6          /* the registered all-reduce callback failed                   */
} mp_status;

/* ----------------------------------------------------------------------------------------
 * a1  State enumeration and transition matrix (host, deterministic)
 * ------------------------------------------------------------------------------------- */

/* |C_n|, the number of correct n-words (Table 1).  No allocation.
 * Errors: MP_ERR_DOMAIN if n < 2 or n > MP_MAX_N. */
mp_status mp_count_words(int n, int64_t *N_out);

/* A(D_n) by Algorithm 1: rows are the words q, columns the words p, both in
 * lexicographic order 0 < 1 < 2 with the first letter (top row of the column) most
 * significant (G5); A_qp = number of zeros of p if p can follow q (P:141-147,
 * readings G2-G4), else MP_INF.
 * The library allocates *A_out (N*N uint16_t, row-major, host memory); the caller
 * releases it with mp_free().  Errors: MP_ERR_DOMAIN (n outside [2, MP_MAX_N], NULL),
 * MP_ERR_RESOURCE (host allocation of 2*N*N bytes failed). */
mp_status build_transition_matrix(int n, uint16_t **A_out, int64_t *N_out);

/* Same matrix written into a caller-owned host buffer of exactly N*N entries (N from
 * mp_count_words).  Errors as above, plus MP_ERR_DOMAIN if N does not match. */
mp_status build_transition_matrix_into(int n, uint16_t *A, int64_t N);

/* Releases memory returned by the library (NULL is a no-op). */
void mp_free(void *p);

/* ----------------------------------------------------------------------------------------
 * a3  (min,+) product ((A x B)_ij = min_k (a_ik + b_kj))
 * ------------------------------------------------------------------------------------- */

/* C = A x B with A M x K, B K x N, C M x N; contiguous row-major HOST buffers, caller
 * owned.  The library stages A and B to the current device, runs the sm_100a DPX kernel,
 * and copies C back.  Errors: MP_ERR_DOMAIN (dims <= 0, NULL, C overlapping A or B),
 * MP_ERR_RANGE, MP_ERR_RESOURCE, MP_ERR_CUDA. */
mp_status minplus_mul(const uint16_t *A, const uint16_t *B, uint16_t *C, int64_t M,
                      int64_t K, int64_t N);

/* Device-pointer variant (e.g. torch tensors' data_ptr()): dA (M x K, pitch lda),
 * dB (K x N, pitch ldb), dC (M x N, pitch ldc) live on the current device, in the
 * boundary encoding above.  Asynchronous on `stream` (a cudaStream_t; NULL = legacy
 * default stream) except that a range violation is reported synchronously (the call
 * synchronises `stream` once to read the range flag).  Scratch buffers are owned by the
 * library and reused across calls.  Errors as minplus_mul. */
mp_status minplus_mul_device(const uint16_t *dA, int64_t lda, const uint16_t *dB, int64_t ldb,
                             uint16_t *dC, int64_t ldc, int64_t M, int64_t K, int64_t N,
                             void *stream);

/* NEXT-4: general products through the same kernel.
 *   minplus_mul_strided_batched_device: C_b = A_b x B_b for b < batch, with A_b = dA +
 *     b*strideA (elements; likewise B_b, C_b; a stride may be 0 to reuse one operand), each as
 *     in minplus_mul_device; every kernel runs once for all items (the batch index is the grid's
 *     z dimension; items are taken in chunks of at most 8 GB of scratch), on `stream`.  Errors as minplus_mul_device, plus MP_ERR_DOMAIN for batch <= 0, a negative
 *     stride, C matrices overlapping each other or any A_b / B_b.
 *   minplus_closure: D = (I (+) W)^(2^t) with 2^t >= N-1 (t squarings; *squarings_out = t if
 *     not NULL): for a weighted adjacency W (N x N host, boundary encoding, W_ij = arc
 *     length) the all-pairs shortest path lengths, +inf if unreachable, path lengths >= 0x7FFF
 *     saturating to +inf (G6).  I (+) W = W with a zero diagonal.  Host buffers, caller-owned.
 *     Sharded over the ranks like minplus_mul when an all-gather is registered.
 *     Errors: MP_ERR_DOMAIN (NULL, N <= 0, D overlapping W), MP_ERR_RANGE, MP_ERR_RESOURCE,
 *     MP_ERR_CUDA. */
mp_status minplus_mul_strided_batched_device(const uint16_t *dA, int64_t lda, int64_t strideA,
                                             const uint16_t *dB, int64_t ldb, int64_t strideB,
                                             uint16_t *dC, int64_t ldc, int64_t strideC, int64_t M,
                                             int64_t K, int64_t N, int64_t batch, void *stream);
mp_status minplus_closure(const uint16_t *W, int64_t N, uint16_t *D, int32_t *squarings_out);

/* ----------------------------------------------------------------------------------------
 * a3-a5  Power sequence until it is quasi-periodic
 * ------------------------------------------------------------------------------------- */

typedef struct {
    int32_t mu;         /* A^{mu+lambda} = offset (x) A^{mu}: mu = the paper's minimal n0   */
    int32_t lambda;     /*   (Alg. 4), lambda = a, offset = b (Theorem 3) */
    int32_t offset;     /*   first repeat up to a constant (G9); 0 if both are all-inf     */
    int32_t k_last;     /* = mu + lambda: the number of powers computed                    */
    int32_t dense_from; /* first k with no +inf entry (0 if none up to k_last)     */
    uint16_t diag_min[MP_MAX_K + 1];    /* diag_min[k] = min_i (A^k)_ii, 1 <= k <= k_last
                                           (Algorithm 5); MP_INF if none     */
    uint64_t fingerprint[MP_MAX_K + 1]; /* H(A^k) = sum_ij s(2i) s(2j+1) x_ij mod 2^64,
                                           s = splitmix64, +inf as 0xFFFF   */
} mp_periodic_result;

/* A^1 = A, A^k = A x A^{k-1} (Algorithm 2, left multiplication G8) for
 * k = 2, 3, ... until the first k with some j < k such that A^k - A^j is constant on the
 * finite entries with an identical +inf pattern (Algorithm 3/4 collapsed into forward
 * first-repeat detection; SURVEY.md section 8(c) "Why first-repeat detection equals
 * Algs. 3/4").  A is an N x N HOST matrix in the boundary encoding.  The power store,
 * products, fingerprints and exact comparisons run on the device; if a distributed
 * context is set (mp_dist_set) every rank passes the same A and owns the column shard
 * mp_shard_range(N, world, rank), and the result is identical on every rank.
 * `out` is caller-owned.  Errors: MP_ERR_DOMAIN (N <= 0, max_k outside [2, MP_MAX_K],
 * NULL), MP_ERR_RANGE, MP_ERR_RESOURCE, MP_ERR_NOT_PERIODIC (out untouched),
 * MP_ERR_CUDA, MP_ERR_COMM. */
mp_status minplus_power_until_periodic(const uint16_t *A, int64_t N, int max_k,
                                       mp_periodic_result *out);

/* Same run with A already resident on the current device: dA is N x N with pitch lda
 * (elements), boundary encoding, device memory owned by the caller and only read.  Work is
 * enqueued on the library stream (see mp_set_stream); the call returns when the result is
 * known.  Errors as minplus_power_until_periodic (MP_ERR_DOMAIN also for lda < N). */
mp_status minplus_power_until_periodic_device(const uint16_t *dA, int64_t lda, int64_t N, int max_k,
                                              mp_periodic_result *out);

/* Parity hook: rows `rows[0..nrows)` of every power A^1..A^kmax, computed by the same
 * device path (staging, product kernel, power store) without the periodicity search.
 * out (caller-owned host buffer) receives kmax*nrows*N entries: out[((k-1)*nrows + r)*N + j]
 * = (A^k)_{rows[r], j}, boundary encoding.  Single device (the distributed context is
 * ignored).  Errors: MP_ERR_DOMAIN (N <= 0, kmax outside [1, MP_MAX_K], nrows <= 0, a row
 * outside [0, N), NULL), MP_ERR_RANGE, MP_ERR_RESOURCE, MP_ERR_CUDA. */
mp_status minplus_power_rows(const uint16_t *A, int64_t N, int kmax, const int64_t *rows, int nrows,
                             uint16_t *out);

/* Parity observer.  While set (fn != NULL), every power run of this process (the matrix
 * sources, the device source and the words source of gamma2_cylinder / mp_gamma2_record; not
 * minplus_power_rows) calls fn(ctx, k, power, N) once per power k = 1 .. k_last, in order, on
 * the calling thread, after A^k and its statistics are computed and before the repeat search
 * looks at it.  power = the WHOLE N x N matrix A^k (Algorithm 2), row-major,
 * boundary encoding (MP_INF = +inf), in a library-owned pinned host buffer valid only during
 * the call; with a symmetry the columns the run does not compute are filled in from their
 * mirrors.  The run itself is unchanged (same kernels, same ring) apart
 * from the extra device buffer of 2 N^2 bytes and the copy.  fn returns 0 to continue; any
 * other value stops the run with MP_ERR_DOMAIN.  fn = NULL clears it.  A run with an observer
 * and a distributed context of world > 1 fails with MP_ERR_DOMAIN (a rank holds only its
 * shard).  Process-wide.  Errors: none (always MP_OK). */
/* Row-inclusion reuse for the transfer matrix (not in the paper).  Row q'
 * of A(D_n) is row q restricted to a subset of its support whenever q' is q with one letter 1
 * turned into a 2 (can-follow, depends on q only through its 0- and 2-positions; the
 * label, only on the column), so every power satisfies (A^k)_q = min((A^k)_q over the
 * extra entries of row q, (A^k)_q' over the parents q') -- the same minimum regrouped.  The SpMM
 * then runs on the extra entries (0.23 of nnz(A) at n = 12) and one fold pass per level of the
 * parent DAG adds the parents' rows.  Used for the words source (gamma2_cylinder) and for matrix
 * sources announced by mp_set_transfer_hint(n): the run then verifies on the device that A is
 * A(D_n) entry by entry (MP_ERR_DOMAIN if not) -- wherever the grouped SpMM runs (N >= 8192
 * with the automatic options).
 *   mp_set_transfer_hint: n = 0 clears; applies to matrix sources of order |C_n|.
 *     Errors: MP_ERR_DOMAIN (n outside {0} u [2, MP_MAX_N]).
 *   mp_set_row_reuse: on = 0 switches the reuse off (same results); default on.  Errors: none.
 * Both process-wide. */
mp_status mp_set_transfer_hint(int n);
mp_status mp_set_row_reuse(int on);

/* Small-N latency path: single-rank power runs of matrices with N <= 256
 * and at most 8192 finite entries, with the automatic kernel choice and no observer, run
 * entirely in one thread-block-cluster launch (products, statistics, repeat search, exact
 * compares; one read of the result).  on = 0 sends them through the general path instead (same
 * results); default on.  Process-wide.  Errors: none. */
mp_status mp_set_small_path(int on);

typedef int (*mp_power_observer_fn)(void *ctx, int k, const uint16_t *power, int64_t N);
mp_status mp_set_power_observer(mp_power_observer_fn fn, void *ctx);

/* ----------------------------------------------------------------------------------------
 * a6  gamma_2(P_n x C_m) (Theorem 2; Theorem 3; solving procedure P:219-222)
 * ------------------------------------------------------------------------------------- */

/* gamma_2 of the cylinder with path order n (2..MP_MAX_N) and cycle length m >= 3.
 * Builds A(D_n), runs minplus_power_until_periodic (max_k = 64) once per n per process
 * (the (mu, lambda, b, diag_min) record is cached), and reads gamma_2 off: diag_min[m] if
 * m <= k_last, else diag_min[m - t*lambda] + t*b with the least t that lands in
 * [mu, k_last].  Errors: MP_ERR_DOMAIN, and those of minplus_power_until_periodic. */
mp_status gamma2_cylinder(int n, int64_t m, int64_t *gamma2_out);

/* The (mu, lambda, b, diag_min, fingerprint) record gamma2_cylinder(n, .) reads from: runs
 * the power sequence of A(D_n) built on the device from the word masks (once per n per
 * process) and copies the cached record to the caller-owned *out.  n = 13 needs the SpMM
 * kernel (default) and about 4 x 34.6 GB of device memory for the power store.
 * Errors: as gamma2_cylinder. */
mp_status mp_gamma2_record(int n, mp_periodic_result *out);

/* Read-off only (host, no device): applies the a6 rule to a result. */
mp_status mp_gamma2_readoff(const mp_periodic_result *r, int64_t m, int64_t *gamma2_out);

/* The closed formula of P:496-502 (NEXT-2): gamma_2(P_n x C_m) = ceil(b*m/a) + alpha[m mod a]
 * for m >= n0 (a = lambda, b = offset, n0 = mu; Theorem 3 solved with the boundary values
 * diag_min[n0 .. n0+a-1], Algorithm 5), plus the cycle lengths 3 <= m < n0 where the formula
 * does not hold ("exceptions", Table 7's starred rows).  Host only.
 * Errors: MP_ERR_DOMAIN (NULL, invalid result, a > MP_MAX_K). */
typedef struct {
    int32_t a, b, n0;
    int32_t r0_k50;                 /* the r0 Algorithm 3 reports with K = 50 (Table 4): the
                                       scan from i = K finds j = K - a first (K >= n0 + a);
                                       -1 if K = 50 < n0 + a                                 */
    int32_t alpha[MP_MAX_K];        /* alpha[k], 0 <= k < a                                   */
    int32_t n_exceptions;
    int64_t exception_m[MP_MAX_K];  /* cycle lengths with gamma_2 != the formula, ascending   */
    int64_t exception_gamma2[MP_MAX_K];
} mp_formula;
mp_status mp_gamma2_formula(const mp_periodic_result *r, mp_formula *out);

/* ----------------------------------------------------------------------------------------
 * Multi-GPU: one process per GPU (torchrun), column shards, a tiny all-reduce per power
 * ------------------------------------------------------------------------------------- */

/* The all-reduce the driver calls once or twice per power on `count` int64 values living
 * in DEVICE memory at dev_buf (already ordered after the library's work on `stream`, which
 * the library synchronises before the call).  op: 0 = SUM (wrapping mod 2^64), 1 = MIN.
 * Returns 0 on success.  The Python binding implements it with torch.distributed over
 * NCCL (NVLink); any MPI-like runtime works. */
typedef int (*mp_allreduce_fn)(void *ctx, int op, int64_t *dev_buf, int64_t count,
                               void *stream);

/* Registers (fn != NULL, world >= 1, 0 <= rank < world) or clears (fn == NULL) the
 * process-wide distributed context used by minplus_power_until_periodic.
 * Errors: MP_ERR_DOMAIN. */
mp_status mp_dist_set(int rank, int world, mp_allreduce_fn fn, void *ctx);

/* The all-gather the general products call when sharded (minplus_mul, minplus_closure): every
 * rank contributes `bytes` bytes at send_dev (DEVICE memory) and receives the world blocks in
 * rank order at recv_dev (world * bytes; already ordered after the library's work on `stream`,
 * which the library synchronises before the call).  Returns 0 on success. */
typedef int (*mp_allgather_fn)(void *ctx, const void *send_dev, void *recv_dev, int64_t bytes, void *stream);

/* Registers (fn != NULL) or clears the all-gather of the distributed context.  With a context
 * of world > 1 and an all-gather, minplus_mul and minplus_closure run column-sharded: every
 * rank passes the same host inputs, rank r computes the column block C[:, J_r] = A (x) B[:, J_r]
 * (J_r = mp_shard_range(N, world, r); A replicated -- the partitioning the paper proposes as
 * future work), the blocks are all-gathered, and every rank's output receives the whole
 * product (the closure all-gathers after every squaring: both of its operands change).
 * Errors: none (always MP_OK). */
mp_status mp_dist_set_allgather(mp_allgather_fn fn, void *ctx);

/* Column shard [*c0, *c1) of rank `rank` among `world` for an N x N power: width
 * w = roundup(ceil(N / world), 8), c0 = min(N, rank*w), c1 = min(N, c0 + w) (the last
 * shard takes the remainder; a shard may be empty when N is tiny).  Pure host function.
 * Errors: MP_ERR_DOMAIN. */
mp_status mp_shard_range(int64_t N, int world, int rank, int64_t *c0, int64_t *c1);

/* Column plan of the SpMM product for a rank computing w columns of an N x N power (DESIGN.md
 * section 6): CTA columns of the run's main width (*main_cols: 1024, 512 or 256 by the grid
 * size, or the mp_set_spmm_width override) and the remainder, rounded up to 64 columns, in up
 * to three narrower CTA columns of 768 / 512 / 256 / 128 / 64 columns (*tail_cols = their
 * total; 0 if none), so *ld (the padded width = the pitch of the powers) exceeds w by less
 * than 64 columns unless a width is forced.  Pure host function
 * (assumes 148 SMs when no device is present).  Errors: MP_ERR_DOMAIN. */
mp_status mp_column_plan(int64_t N, int64_t w, int64_t *ld, int32_t *main_cols, int32_t *tail_cols);

/* ----------------------------------------------------------------------------------------
 * Periodicity bookkeeping (pure host functions; exported so the multi-rank logic is
 * testable without a GPU)
 * ------------------------------------------------------------------------------------- */

/* Per-power statistics after the all-reduce.  Every field is
 * an int64 so that one SUM and one MIN all-reduce carry them: */
typedef struct {
    int64_t fingerprint; /* SUM: canonical linear hash H (the uint64 bits, wrapping)          */
    int64_t inf_count;   /* SUM: number of +inf entries                                      */
    int64_t diag_min;    /* MIN: min_i X_ii (0xFFFF if every diagonal entry is +inf)          */
    int64_t ref;         /* MIN: (t << 16) | x_t of the first finite entry in canonical order
                            t = i*N + j; INT64_MAX if the matrix is all +inf                 */
} mp_power_stats;

/* S(N) = sum_{i,j < N} s(2i) s(2j+1) mod 2^64, s = splitmix64 (the fingerprint of the
 * all-ones matrix). */
uint64_t mp_fingerprint_unit(int64_t N);

/* Candidate test of the forward first-repeat search: returns 1 if A^k may equal
 * c (x) A^j, with c = x_k - x_j taken at the first finite entry (whose position must agree):
 * both powers inf-free and H_k - H_j == c * S(N) (mod 2^64), or both containing +inf with
 * equal counts and equal first-finite positions (the exact comparison decides); both all
 * +inf gives c = 0.  Returns 0 if they certainly differ.  *c_out receives c. */
int mp_repeat_candidate(const mp_power_stats *sk, const mp_power_stats *sj, uint64_t S,
                        int32_t *c_out);

/* ----------------------------------------------------------------------------------------
 * Diagnostics
 * ------------------------------------------------------------------------------------- */

const char *mp_last_error(void); /* thread-local message for the last non-OK status     */
void mp_shutdown(void);          /* frees cached device state and the gamma_2 cache       */
const char *mp_version(void);    /* build string (kernel variant, arch)                   */

/* Number of device kernels launched by this process so far (all entry points). */
int64_t mp_kernel_launches(void);

/* Profiling counters of the last minplus_power_until_periodic call: total milliseconds
 * spent in the product kernel (CUDA events on the library stream), number of product
 * launches, dense-equivalent inner steps (rows*inner*cols summed over launches) and the
 * inner steps actually issued after skipping all-inf A tiles. */
typedef struct {
    double product_ms;        /* sum of product-kernel durations (CUDA events)              */
    int64_t product_launches; /* number of product launches                                 */
    double dense_steps;       /* sum of N * N * w over the launches (dense-equivalent steps) */
    double issued_steps;      /* steps the kernel executed after skipping all-inf A tiles   */
    double total_ms;          /* whole run, first to last operation on the library stream  */
    double setup_ms;          /* of which staging A and building the sparse form (a1-a2)   */
    double stats_ms;          /* sum of the per-power statistics kernel durations (a4)     */
    int64_t h2d_bytes;        /* host -> device bytes copied by the run                    */
    int64_t d2h_bytes;        /* device -> host bytes copied by the run                    */
    int32_t kernel;           /* product kernel used: 0 dense tiles, 1 block-sparse tiles,
                                 2 grouped SpMM, 3 the fused small-N run (product_ms = the
                                 whole run's one launch, statistics included)                */
    int32_t spmm_cols;        /* SpMM CTA width used (256, 512 or 1024 columns; 0 if kernel != 2) */
    int64_t local_cols;       /* columns this rank computes per power (its shard; with a symmetry
                                 a shard of the domain g <= sigma g)                          */
    int64_t ld;               /* pitch of the device powers (local_cols padded to the CTA width) */
    double spmm_ms;           /* of product_ms, the product kernel itself (without the fold
                                 passes of the row-inclusion reuse)                          */
    int32_t row_levels;       /* row-inclusion reuse: levels of the parent DAG (0 = not used)   */
    int64_t row_parents;      /*   and its number of parent links                               */
    double fold_bytes;        /*   algorithmic bytes of one product's fold passes: every folded
                                   row read and written once, each distinct parent row of a
                                   level read once by that level's pass (x ld x 2 bytes)         */
} mp_profile;
mp_status mp_last_profile(mp_profile *out);

/* Stream for the power runs on the current device (a cudaStream_t, e.g. torch's current
 * stream, so that caller-side CUDA events bracket a run); NULL restores the library's own
 * non-blocking stream, so the legacy default stream is passed as cudaStreamLegacy ((void *)1;
 * the Python binding maps torch's default stream, handle 0, to it).  Errors: MP_ERR_CUDA if
 * no device. */
mp_status mp_set_stream(void *stream);

/* Tuning knobs (process-wide; defaults in DESIGN.md).  sparsity selects the product kernel
 * of the power runs: 0 = dense 128x256x32 tiles over all of A; 1 = the same kernel skipping
 * the all-inf tiles of A; 2 = the grouped (8-row) SpMM kernel over A's finite entries;
 * -1 = automatic (the default: SpMM when it issues fewer than 60 % of the tile kernel's
 * steps).  All are exact (an all-inf term never lowers a minimum).  device_budget_bytes caps
 * the power store (0 = min(48 GiB, 90 % of free device memory)).  Errors: MP_ERR_DOMAIN. */
mp_status mp_set_options(int sparsity, int64_t device_budget_bytes);

/* Symmetry of A (not in the paper): an involution sigma of [0, N) with
 * A[sigma i][sigma j] = A[i][j] for all i, j.  Every power then has the same symmetry and
 * column j of A^k depends only on column j of A^{k-1}, so the power runs compute only the
 * columns g <= sigma(g) (about half) and derive every statistic of the full matrix from them;
 * all outputs are those of the full computation.
 *   mp_set_symmetry: hint for the matrix sources of size N (host array of N int32, copied;
 *     NULL or N <= 0 clears it).  Each run verifies it on the device and fails with
 *     MP_ERR_DOMAIN if some finite A_ij != A_(sigma i, sigma j).  Errors: MP_ERR_DOMAIN (not
 *     an involution).
 *   mp_set_word_symmetry: the words source (gamma2_cylinder, mp_gamma2_record) uses the word
 *     reversal (the reflection of the path P_n, which the can-follow rule P:141-147 and the
 *     labels P:152 respect) unless switched off (on = 0); default on.
 *   mp_word_reversal: sigma_out[i] = index of the reversed word i in A(D_n) (N = its order,
 *     caller-owned buffer).  Errors: MP_ERR_DOMAIN (n outside [2, MP_MAX_N], N mismatch). */
mp_status mp_set_symmetry(const int32_t *sigma, int64_t N);
mp_status mp_set_word_symmetry(int on);
mp_status mp_word_reversal(int n, int32_t *sigma_out, int64_t N);

/* Row grouping of the SpMM kernel (sparsity 2): 0 = groups of 4 consecutive rows; 1 = rows
 * grouped greedily by support overlap in windows of 256 rows (fewer issued steps, same
 * product); -1 = automatic (the default: greedy from N >= 8192).
 * Process-wide.  Errors: MP_ERR_DOMAIN. */
mp_status mp_set_grouping(int mode);

/* CTA width of the SpMM kernel (sparsity 2), in columns: 256 (4 packed column pairs per
 * lane, 3 CTAs per SM), 512 (8 pairs per lane, 3 CTAs per SM), 1024 (16 pairs per lane, 2 CTAs
 * per SM: half the per-entry overhead, half the CTAs) for every CTA, the power pitch padded to a
 * multiple of it; the negative values -256, -512, -1024 set the main width but keep the
 * narrower CTA columns for the remainder (mp_column_plan); 0 = automatic (the default: main
 * width 1024 when the grid still has at least 24 CTAs per SM, i.e. n >= 11 for A(D_n); else 512
 * when that grid has at least 8 CTAs per SM, i.e. n = 10; else 256; plus the remainder
 * columns).  Same product either way.  Process-wide.  Errors: MP_ERR_DOMAIN. */
mp_status mp_set_spmm_width(int cols);

#ifdef __cplusplus
}
#endif
#endif /* MINPLUS_H */
