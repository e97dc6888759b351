// Host launchers of the device kernels in mp_kernels.cu (internal).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "mp_internal.h"

namespace mp {

// C[Mp][ldc] = AT2 (x) X over Kp inner steps, for the column tiles [0, ncols_p).
// kt_ptr/kt_idx: optional per-row-tile list of l-tiles with a finite A entry.
cudaError_t launch_minplus(const uint32_t *AT2, int64_t lda, const uint16_t *X, int64_t ldx, uint16_t *C,
                           int64_t ldc, int64_t Mp, int64_t ncols_p, int64_t Kp, const int32_t *kt_ptr,
                           const int32_t *kt_idx, cudaStream_t s);
cudaError_t launch_stats(const uint16_t *X, int64_t ld, int64_t N, int64_t c0, int64_t w,
                         unsigned long long *out, cudaStream_t s);
cudaError_t launch_compare(const uint16_t *Y, const uint16_t *Z, int64_t ld, int64_t N, int64_t w, int32_t c,
                           unsigned long long *out, cudaStream_t s);
cudaError_t launch_encode(const uint16_t *src, int64_t lds, int64_t rows, int64_t cols, uint16_t *dst,
                          int64_t ldd, int64_t rows_p, int *range_flag, cudaStream_t s);
cudaError_t launch_make_at2(const uint16_t *A, int64_t lda, int64_t M, int64_t K, uint32_t *AT2, int64_t Mp,
                            int64_t Kp, int *range_flag, cudaStream_t s);
cudaError_t launch_build_from_words(const WordMask *words, int64_t N, int n, uint32_t *AT2, int64_t Np,
                                    cudaStream_t s);
cudaError_t launch_x1_from_at2(const uint32_t *AT2, int64_t Np, int64_t c0, int64_t w, uint16_t *X1,
                               int64_t ldx, cudaStream_t s);
cudaError_t launch_decode(const uint16_t *src, int64_t lds, int64_t rows, int64_t cols, uint16_t *dst,
                          int64_t ldd, cudaStream_t s);
// Grouped sparse form of A for the SpMM product (see k_spmm8).
struct SparseA {
    const int32_t *L = nullptr;    // concatenated per-tile union lists of l
    const int64_t *tptr = nullptr; // [Np/128 + 1] offsets into L
    const int32_t *epos = nullptr; // per entry: position of its l in its tile's union list
    const uint4 *ea = nullptr;     // per entry: 8 duplicated values (2 x uint4)
    const int64_t *eptr = nullptr; // [Np/8 + 1] offsets of each group's entries
};
cudaError_t launch_spmm(const SparseA &sa, const uint16_t *X, int64_t ldx, uint16_t *C, int64_t ldc, int64_t Mp,
                        int64_t ncols_p, cudaStream_t s);
cudaError_t sparse_masks(const uint32_t *AT2, int64_t Np, uint8_t *m8, cudaStream_t s);
cudaError_t sparse_tile_union(const uint8_t *m8, int64_t Np, const int64_t *tptr, int32_t *tcnt, int32_t *L,
                              int32_t *posmap, cudaStream_t s);
cudaError_t sparse_group_entries(const uint8_t *m8, const uint32_t *AT2, int64_t Np, const int64_t *eptr,
                                 const int32_t *posmap, int32_t *gcnt, int32_t *epos, uint4 *ea, cudaStream_t s);
cudaError_t scan_counts(const int32_t *cnt, int64_t n, int64_t *out, cudaStream_t s);
cudaError_t launch_unit_sum(int64_t N, unsigned long long *out, cudaStream_t s);
cudaError_t launch_tile_occupancy(const uint32_t *AT2, int64_t Mp, int64_t Kp, uint8_t *occ, cudaStream_t s);

} // namespace mp
