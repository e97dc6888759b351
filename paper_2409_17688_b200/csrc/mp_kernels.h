// Host launchers of the device kernels in mp_kernels.cu (internal).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "mp_internal.h"

namespace mp {

// C[Mp][ldc] = AT2 (x) X over Kp inner steps, for the column tiles [0, ncols_p).
// kt_ptr/kt_idx: optional per-row-tile list of l-tiles with a finite A entry.
// batch > 1: items b < batch at AT2 + b sA, X + b sX, C + b sC, all in one launch (grid z).
cudaError_t launch_minplus(const uint32_t *AT2, int64_t lda, const uint16_t *X, int64_t ldx, uint16_t *C,
                           int64_t ldc, int64_t Mp, int64_t ncols_p, int64_t Kp, const int32_t *kt_ptr,
                           const int32_t *kt_idx, cudaStream_t s, int batch = 1, int64_t sA = 0, int64_t sX = 0,
                           int64_t sC = 0);
cudaError_t launch_stats(const uint16_t *X, int64_t ld, int64_t N, int64_t c0, int64_t w,
                         unsigned long long *out_sum, unsigned long long *out_min, cudaStream_t s);
cudaError_t launch_compare(const uint16_t *Y, const uint16_t *Z, int64_t ld, int64_t N, int64_t w, int32_t c,
                           unsigned long long *out, cudaStream_t s);
cudaError_t launch_encode(const uint16_t *src, int64_t lds, int64_t rows, int64_t cols, uint16_t *dst,
                          int64_t ldd, int64_t rows_p, int *range_flag, cudaStream_t s, int batch = 1,
                          int64_t ss = 0, int64_t sd = 0);
cudaError_t launch_make_at2(const uint16_t *A, int64_t lda, int64_t M, int64_t K, uint32_t *AT2, int64_t Mp,
                            int64_t Kp, int *range_flag, cudaStream_t s, int batch = 1, int64_t sa = 0,
                            int64_t sat = 0);
cudaError_t launch_build_from_words(const WordMask *words, int64_t N, int n, uint32_t *AT2, int64_t Np,
                                    cudaStream_t s);
cudaError_t launch_x1_from_at2(const uint32_t *AT2, int64_t Np, int64_t c0, int64_t w, uint16_t *X1,
                               int64_t ldx, cudaStream_t s);
// C[i][r w + j] = G[r][i][j]: world all-gathered M x w column blocks into the M x N matrix C.
cudaError_t launch_unshard(const uint16_t *G, int world, int64_t M, int64_t w, int64_t N, uint16_t *C, int64_t ldc,
                           cudaStream_t s);
// X[i][i] = 0 for i < n.
cudaError_t launch_set_diag_zero(uint16_t *X, int64_t ld, int64_t n, cudaStream_t s);
cudaError_t launch_decode(const uint16_t *src, int64_t lds, int64_t rows, int64_t cols, uint16_t *dst,
                          int64_t ldd, cudaStream_t s, int batch = 1, int64_t ss = 0, int64_t sd = 0);
// Small-N latency path (mp_small.cu): the whole power-until-periodic run in one cluster launch.
// sigma (may be null): symmetry hint verified on the way (status 1 if violated).
// out[]: status (0 ok, 1 hint violated, 2 range, 4 not periodic, -1 more than max_nnz finite
// entries), mu, lambda,
// offset, k_last, dense_from, then diag_min[k] at out[6 + k] and fingerprint[k] at
// out[6 + (max_k + 1) + k], then 4 clock64 phase sums.  hist: (max_k + 1) x N x (64 * ctas) u16.
constexpr int kSmallMaxN = 256;
int small_run_ctas(int64_t N);
cudaError_t launch_small_run(const uint16_t *A, int64_t lda, int64_t N, int max_k, int max_nnz, const int32_t *sigma,
                             uint16_t *hist, uint64_t S, long long *out, cudaStream_t s);
// out (N x N, boundary encoding) = the whole power from the local columns of X: column g is
// local column loc[g] if loc[g] >= 0, else X_(sigma i, loc[sigma g]) (sigma may be null only if
// every column is local).
cudaError_t launch_unfold(const uint16_t *X, int64_t ld, int64_t N, const int32_t *loc, const int32_t *sigma,
                          uint16_t *out, cudaStream_t s);
// Grouped sparse form of A for the SpMM product (see k_spmm in mp_kernels.cu).
struct SparseA {
    const int32_t *L = nullptr;    // concatenated per-tile (32-row) ordered union lists of l
    const int64_t *tptr = nullptr; // [Mt + 1] offsets into L
    const int64_t *tch = nullptr;  // [Mt + 1] first chunk of each tile
    const int64_t *eoff = nullptr; // [chunks * 8 + 1] entry offsets per (chunk, group)
    const uint4 *E = nullptr;      // entries, 3 x uint4 each
    const int32_t *rows = nullptr; // group slot -> row of A (null: identity)
};
// Device buffers of the sparse form (owned by the caller; allocated through `alloc`).
struct SparseWork {
    uint8_t *m8 = nullptr;
    int32_t *tcnt = nullptr, *nch = nullptr, *L = nullptr, *chunk_tile = nullptr, *ecnt = nullptr;
    int64_t *tptr = nullptr, *tch = nullptr, *eoff = nullptr;
    uint4 *E = nullptr;
    int32_t *rows = nullptr; // row grouping (null: consecutive rows)
    uint32_t *bits = nullptr; // support bitsets (grouped path)
    int64_t *off = nullptr;   // row lists of A's support (grouped path): CSR offsets ...
    int32_t *idx = nullptr;   // ... and column indices
    int group_rows = 0;      // rows per group: issued steps = entries * group_rows * ld
    int cols = 512;          // set by the caller: the k_spmm CTA width the entries are built for
    int64_t total_union = 0, total_chunks = 0, entries = 0;
};
// cols = the CTA width, 512 or 1024 (ncols_p must be a multiple of it): spmm_cols(Np, w) picks
// it per run from the grid size (or the mp_set_spmm_width override in g_spmm_width).
int spmm_cols(int64_t Np, int64_t w);
extern int g_spmm_width;
// Column plan of one SpMM product over w local columns: CTA columns of the run's main width
// (spmm_cols) and, for the remainder rounded up to 64 columns, up to three narrower CTA columns
// (768, 512, 256, 128, 64), so a shard is padded by less than 64 columns instead of up to
// main - 1.
// ld = the padded width = the pitch of the powers.
struct SpmmPlan {
    struct Seg {
        int64_t col0; // first local column
        int cols;     // CTA width (1024, 768, 512, 256, 128 or 64)
        int64_t ncols; // columns of this segment (a multiple of cols)
    };
    Seg seg[4];
    int nseg = 0;
    int main_cols = 0;
    int64_t ld = 0;
};
SpmmPlan spmm_plan(int64_t Np, int64_t w);
// One launch per segment of the plan (*launches counts them).
cudaError_t launch_spmm(const SparseA &sa, const SpmmPlan &P, const uint16_t *X, int64_t ldx, uint16_t *C,
                        int64_t ldc, int64_t Mp, cudaStream_t s, int *launches);
// Row-inclusion reuse for A(D_n) (mp_dag.cu): parents of row q = the
// words q with one letter 0 or 1 turned into 2 (their rows are restrictions of row q); rows by
// level.
struct RowDag {
    int64_t *off = nullptr;     // [N + 1] parent lists (CSR)
    int32_t *idx = nullptr;     // parents
    int32_t *level = nullptr;   // [N] 0 without parents, else 1 + max level of the parents
    int32_t *lrows = nullptr;   // [N] rows grouped by level
    int64_t *lptr_dev = nullptr;
    int *bad = nullptr;         // set by launch_extra_bits if a parent's support is not a subset
    std::vector<int64_t> lptr;  // [levels + 1] level offsets into lrows (host copy)
    int levels = 0;
    int64_t parents = 0;
    // the folds' algorithmic traffic in rows per product: every folded row read and written once,
    // each distinct parent row of a level read once by that level's launch
    int64_t fold_rows = 0;
};
cudaError_t build_row_dag(const WordMask *words, int64_t N, int n, RowDag &d, cudaStream_t s,
                          cudaError_t (*alloc)(void **, size_t, void *), void *actx, int64_t *launches);
// ebits = bits minus the union of the parents' bits, row by row (N x nw words each)
cudaError_t launch_extra_bits(const uint32_t *bits, int64_t nw, int64_t N, const RowDag &d, uint32_t *ebits,
                              cudaStream_t s);
// C_q = min(C_q, C_p) over the parents p, level by level (levels 1 .. levels-1), ncols columns
cudaError_t launch_folds(const RowDag &d, uint16_t *C, int64_t ldc, int64_t ncols, cudaStream_t s, int *launches);
// group: form the row groups with k_group_greedy (else groups are consecutive rows).
// A: the matrix source itself (row-major, boundary encoding, range-checked by launch_check_a).
// pre_bits (may be null): A's support bitsets from launch_check_a (N x ceil(N/32) words).
// dag (may be null; needs group): build the form on the extra entries of each row only.
cudaError_t build_sparse_form(const uint16_t *A, int64_t lda, int64_t N, int64_t Np, bool group,
                              const uint32_t *pre_bits, SparseWork &w, cudaStream_t s,
                              cudaError_t (*alloc)(void **, size_t, void *), void *actx, int64_t *launches,
                              const RowDag *dag = nullptr);
cudaError_t build_sparse_form_words(const WordMask *words, int64_t N, int n, int64_t Np, bool group, SparseWork &w,
                                    cudaStream_t s, cudaError_t (*alloc)(void **, size_t, void *), void *actx,
                                    int64_t *launches, const RowDag *dag = nullptr);
// gcol (may be null): the global column of each local column (else c0 + j).
cudaError_t launch_x1_from_words(const WordMask *words, int64_t N, int n, int64_t Np, int64_t c0, const int32_t *gcol,
                                 int64_t w, uint16_t *X1, int64_t ldx, cudaStream_t s);
// X_1 from the row lists of A: +inf everywhere, then each finite a_il with loc[l] >= 0 at
// X1[i][loc[l]] (value from A, or the label zeros(l) of the words source if A is null).
cudaError_t launch_x1_csr(const int64_t *off, const int32_t *idx, int64_t N, const uint16_t *A, int64_t lda,
                          const WordMask *words, const int32_t *loc, uint16_t *X1, int64_t ldx, int64_t Np,
                          cudaStream_t s);
// X_1 from A's support bitsets (from launch_check_a): +inf everywhere, then each finite a_il
// with loc[l] >= 0 at X1[i][loc[l]] (two launches).
cudaError_t launch_x1_bits(const uint32_t *bits, int64_t N, const uint16_t *A, int64_t lda, const int32_t *loc,
                           uint16_t *X1, int64_t ldx, int64_t Np, cudaStream_t s);
// X_1 on a column list: dst[i][j] = enc(src[i][gcol[j]]).
cudaError_t launch_encode_cols(const uint16_t *src, int64_t lds, int64_t rows, const int32_t *gcol, int64_t w,
                               uint16_t *dst, int64_t ldd, int64_t rows_p, cudaStream_t s);
// Statistics of the full matrix from its columns gcol[0..w) under the symmetry sigma.
// rw / rwm: the row weights of launch_row_weights.
// tcs (may be null): {fingerprint, nonzero if the power holds +inf} of the tensor-core pass
// (launch_fp_tc) for this power; the kernel adds that fingerprint instead of hashing, and
// without +inf finds the diagonal minimum and first finite key directly (one column per
// thread), else it scans the power for them and the +inf count.
cudaError_t launch_stats_sym(const uint16_t *X, int64_t ld, int64_t N, const int32_t *gcol, const int32_t *sigma,
                             const uint64_t *rw, const uint64_t *rwm, int64_t w, unsigned long long *out_sum,
                             unsigned long long *out_min, cudaStream_t s, const unsigned long long *tcs = nullptr);
// The fingerprint of a power on its w local columns (column jj = gcol[jj], mirrors sigma) by
// 8-bit integer tensor-core MMAs (mp_fptc.cu), plus a nonzero count if it holds +inf, added into
// tcs[0], tcs[1] (zeroed by the caller).  prev: the previous power's tcs (null for the first
// power): +inf is remapped to 0xFFFF only if prev is null or held +inf; otherwise a power with
// +inf gets bit 63 of tcs[1] (fingerprint void).  wfrag: the column weights' byte fragments
// from launch_fp_tc_weights (ld / 32 chunks x 32 lanes x uint4).
cudaError_t launch_fp_tc_weights(const int32_t *gcol, const int32_t *sigma, int64_t w, int64_t ld, uint4 *wfrag,
                                 cudaStream_t s);
cudaError_t launch_fp_tc(const uint16_t *X, int64_t ld, int64_t N, int64_t w, const uint4 *wfrag, const uint64_t *rw,
                         const uint64_t *rwm, unsigned long long *tcs, cudaStream_t s, const unsigned long long *prev);
// rw[i] = s(2i), rwm[i] = s(2 sigma i) for i < N.
cudaError_t launch_row_weights(int64_t N, const int32_t *sigma, uint64_t *rw, uint64_t *rwm, cudaStream_t s);
// Range check of a row-major A (flag set if an entry lies in (0x7FFE, 0xFFFF)) and, if occ is
// not null, the occupancy of its 128 x 32 tiles (occ zeroed by the caller).
// If sigma is not null, sym_flag is set when some finite A_ij != A_(sigma i, sigma j).
// If bits is not null it receives A's support bitsets (bit b of bits[i * ceil(N/32) + k] =
// A_(i, 32k + b) finite).
// If words is not null, *xfer_flag is set unless A equals A(D_n) entry by entry (the transfer
// hint, verified in the same pass).
cudaError_t launch_check_a(const uint16_t *A, int64_t lda, int64_t N, int64_t Np, uint8_t *occ, int *range_flag,
                           const int32_t *sigma, int *sym_flag, uint32_t *bits, cudaStream_t s,
                           const WordMask *words = nullptr, int n = 0, int *xfer_flag = nullptr);
cudaError_t launch_tile_occupancy(const uint32_t *AT2, int64_t Mp, int64_t Kp, uint8_t *occ, cudaStream_t s);

} // namespace mp
