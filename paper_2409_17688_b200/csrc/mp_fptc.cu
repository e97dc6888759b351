// The a4 fingerprint on the tensor cores (round 2; DESIGN.md section 5 "Fingerprint on the
// tensor cores").  Product code only; shares nothing with oracle/.
//
// With the symmetry the fingerprint of a power is a rank-2 bilinear form
// over the stored columns:
//     H = sum_i sum_jj x_(i,jj) (a_i b_jj + a'_i b'_jj)  (mod 2^64),
// a_i = s(2i), a'_i = s(2 sigma i), b_jj = s(2g+1), b'_jj = s(2 sigma g + 1) (0 if sigma g = g),
// g = gcol[jj], x with +inf counted as 0xFFFF.  That is a matrix-vector product X b followed by
// a dot product with a: a real contraction.  Split x = x0 + 256 x1 into two byte planes and
// b = sum_t b_t 256^t into its 8 bytes; then
//     (X b)_i = sum_{p=0,1} sum_{t=0..7} 256^(p+t) (X_p B)_(i,t)  (mod 2^64),
// where X_p B (rows x 32-column chunks of u8 times 32 x 8 byte matrices) is exact in 32 bits:
// each term is at most 255^2 and a row has fewer than 66052 columns.  The products run as
// mma.sync m16n8k32 u8 x u8 -> s32 (IMMA on sm_100a): one warp owns 16 rows, walks 32-column
// chunks two at a time, loads its 4 x 4 u16 of X per chunk, splits the bytes with PRMT and
// issues 4 MMAs (2 planes x {b, b'}); about 1.5 instructions per entry (the CUDA-core
// k_stats_sym needs about 20).  A power with +inf entries (only the first powers of A(D_n)) is
// flagged: k_stats_sym then scans it for the other statistics, without hashing.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "mp_internal.h"
#include "mp_kernels.h"

namespace mp {

namespace {

#ifndef MP_FPTC_CHUNKS
#define MP_FPTC_CHUNKS 2
#endif
#ifndef MP_FPTC_MINB
#define MP_FPTC_MINB 3
#endif
constexpr int kFpChunks = MP_FPTC_CHUNKS; // 32-column chunks in flight per warp

__device__ __forceinline__ void imma(int (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1)
{
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};\n"
                 : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// wfrag[chunk][lane] = the B fragments of lane (groupID n = lane / 4 = byte index, k = 4 (lane % 4)
// + i): {bytes n of b for columns 32 chunk + 4 (lane % 4) + i, the same + 16, then b'}
__global__ void k_fp_tc_weights(const int32_t *__restrict__ gcol, const int32_t *__restrict__ sigma, int64_t w,
                                int64_t nchunks, uint4 *__restrict__ wfrag)
{
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nchunks * 32;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t chunk = t >> 5;
        const int lane = (int)(t & 31), n = lane >> 2, tig = lane & 3;
        uint32_t r[4] = {0, 0, 0, 0};
#pragma unroll
        for (int half = 0; half < 2; ++half)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int64_t jj = chunk * 32 + 4 * tig + i + 16 * half;
                uint64_t b = 0, bm = 0;
                if (jj < w) {
                    const int32_t g = gcol[jj], m = sigma[g];
                    b = mix64(2 * (uint64_t)g + 1);
                    bm = m != g ? mix64(2 * (uint64_t)m + 1) : 0;
                }
                r[half] |= (uint32_t)((b >> (8 * n)) & 0xFFu) << (8 * i);
                r[2 + half] |= (uint32_t)((bm >> (8 * n)) & 0xFFu) << (8 * i);
            }
        wfrag[t] = make_uint4(r[0], r[1], r[2], r[3]);
    }
}

// One 32-column chunk: the lane's 4 x 4 u16 of X (rows r0, r1; columns 4 tig .. and + 16),
// the column weights' B fragments, and the chunk's 4 MMAs.  +inf entries become 0xFFFF, and
// their presence is flagged (k_stats_sym then still scans for the +inf count and the first
// finite entry).
struct Chunk {
    uint2 q00, q10, q01, q11;
    uint4 wf;
};

__device__ __forceinline__ void load_chunk(Chunk &h, const uint16_t *x0, const uint16_t *x1, int64_t col,
                                           const uint4 *wf)
{
    h.q00 = *reinterpret_cast<const uint2 *>(x0 + col);
    h.q10 = *reinterpret_cast<const uint2 *>(x1 + col);
    h.q01 = *reinterpret_cast<const uint2 *>(x0 + col + 16);
    h.q11 = *reinterpret_cast<const uint2 *>(x1 + col + 16);
    h.wf = *wf;
}

// +inf (0x7FFF) counts as 0xFFFF (FIX): q | (cmp & 0x80008000); without FIX the comparison
// only flags the chunk
template <bool FIX>
__device__ __forceinline__ void fix_inf(uint32_t &q, uint32_t &any)
{
    const uint32_t c = __vcmpeq2(q, 0x7FFF7FFFu);
    if (FIX) q |= c & 0x80008000u;
    any |= c;
}

template <bool FIX>
__device__ __forceinline__ void mma_chunk(int (&acc)[4][4], Chunk h, uint32_t &anyinf)
{
    fix_inf<FIX>(h.q00.x, anyinf), fix_inf<FIX>(h.q00.y, anyinf), fix_inf<FIX>(h.q10.x, anyinf);
    fix_inf<FIX>(h.q10.y, anyinf), fix_inf<FIX>(h.q01.x, anyinf), fix_inf<FIX>(h.q01.y, anyinf);
    fix_inf<FIX>(h.q11.x, anyinf), fix_inf<FIX>(h.q11.y, anyinf);
    // A fragments: a0 = (row n, cols 4 tig..), a1 = (row n + 8, ..), a2 / a3 = cols + 16
    const uint32_t lo[4] = {__byte_perm(h.q00.x, h.q00.y, 0x6420), __byte_perm(h.q10.x, h.q10.y, 0x6420),
                            __byte_perm(h.q01.x, h.q01.y, 0x6420), __byte_perm(h.q11.x, h.q11.y, 0x6420)};
    const uint32_t hi[4] = {__byte_perm(h.q00.x, h.q00.y, 0x7531), __byte_perm(h.q10.x, h.q10.y, 0x7531),
                            __byte_perm(h.q01.x, h.q01.y, 0x7531), __byte_perm(h.q11.x, h.q11.y, 0x7531)};
    imma(acc[0], lo, h.wf.x, h.wf.y);
    imma(acc[1], lo, h.wf.z, h.wf.w);
    imma(acc[2], hi, h.wf.x, h.wf.y);
    imma(acc[3], hi, h.wf.z, h.wf.w);
}

// D fragment: d0, d1 = (row n, bytes 2 tig, 2 tig + 1), d2, d3 = (row n + 8, same bytes).
// u = sum_{p, t} 256^(p + t) D_p[t] over this lane's two bytes, then over the group's four
// lanes (all eight bytes): sums of 32-bit values as unsigned, mod 2^64; times the row weights.
__device__ __forceinline__ void tile_hash(const int (&acc)[4][4], int tig, int64_t r0, int64_t r1, bool v0, bool v1,
                                          const uint64_t *__restrict__ rw, const uint64_t *__restrict__ rwm,
                                          unsigned long long &hacc)
{
    uint64_t u[2] = {0, 0}, um[2] = {0, 0};
#pragma unroll
    for (int rr = 0; rr < 2; ++rr)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int t = 2 * tig + e;
            const int d = 2 * rr + e;
            u[rr] += ((uint64_t)(uint32_t)acc[0][d] << (8 * t)) + ((uint64_t)(uint32_t)acc[2][d] << (8 * t + 8));
            um[rr] += ((uint64_t)(uint32_t)acc[1][d] << (8 * t)) + ((uint64_t)(uint32_t)acc[3][d] << (8 * t + 8));
        }
#pragma unroll
    for (int o = 1; o < 4; o <<= 1)
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
            u[rr] += __shfl_xor_sync(0xFFFFFFFFu, u[rr], o);
            um[rr] += __shfl_xor_sync(0xFFFFFFFFu, um[rr], o);
        }
    if (tig == 0) {
        if (v0) hacc += rw[r0] * u[0] + rwm[r0] * um[0];
        if (v1) hacc += rw[r1] * u[1] + rwm[r1] * um[1];
    }
}

// The warp's fingerprint part and +inf flag into tcs: +inf present counts the warp; without the
// remapping (FIX) the fingerprint is void (bit 63; the counts never reach it)
template <bool FIX>
__device__ __forceinline__ void warp_flush(unsigned long long hacc, uint32_t anyinf, unsigned long long *tcs)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        hacc += __shfl_xor_sync(0xFFFFFFFFu, hacc, o);
        anyinf |= __shfl_xor_sync(0xFFFFFFFFu, anyinf, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (hacc) atomicAdd(tcs + 0, hacc);
        if (anyinf) {
            atomicAdd(tcs + 1, 1ull);
            if (!FIX) atomicOr(tcs + 1, 1ull << 63);
        }
    }
}

// Work item = (16-row tile, column part): the part's chunks [c0, c1).  Rows >= N and columns
// >= w read as 0 (the last tile / chunk); the other chunks go two at a time (the next pair's
// loads are in flight while the current pair's MMAs issue).
template <bool FIX>
__device__ __forceinline__ void fp_tc_body(const uint16_t *__restrict__ X, int64_t ld, int64_t N, int64_t w,
                                           const uint4 *__restrict__ wfrag, const uint64_t *__restrict__ rw,
                                           const uint64_t *__restrict__ rwm, int64_t ntiles, int64_t nparts,
                                           int64_t chunks_per_part, int64_t nchunks, unsigned long long *__restrict__ tcs,
                                           const uint16_t *zero_row)
{
    const int lane = threadIdx.x & 31, n = lane >> 2, tig = lane & 3;
    unsigned long long hacc = 0;
    uint32_t anyinf = 0;
    const int64_t items = ntiles * nparts, nfull = w / 32; // chunks without padding columns
    for (int64_t it = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < items;
         it += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t tile = it / nparts, part = it - tile * nparts;
        const int64_t r0 = tile * 16 + n, r1 = r0 + 8; // this lane's two rows
        const bool v0 = r0 < N, v1 = r1 < N;
        const int64_t ca = part * chunks_per_part, cb = min(nchunks, ca + chunks_per_part);
        const int64_t cfull = min(cb, nfull);
        int acc[4][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}, {0, 0, 0, 0}, {0, 0, 0, 0}}; // {p0 b, p0 b', p1 b, p1 b'}
        // rows past N read the zero row (shared memory, through generic pointers)
        const uint16_t *x0 = v0 ? X + r0 * ld : zero_row, *x1 = v1 ? X + r1 * ld : zero_row;
        const int64_t s0 = v0 ? 1 : 0, s1 = v1 ? 1 : 0; // column stride multiplier (0: the zero row)
        int64_t c = ca;
        if (tile * 16 + 16 <= N) { // warp-uniform (mma.sync needs the whole warp)
            for (; c + kFpChunks <= cfull; c += kFpChunks) {
                Chunk h[kFpChunks];
#pragma unroll
                for (int q = 0; q < kFpChunks; ++q)
                    load_chunk(h[q], x0, x1, (c + q) * 32 + 4 * tig, wfrag + (c + q) * 32 + lane);
#pragma unroll
                for (int q = 0; q < kFpChunks; ++q) mma_chunk<FIX>(acc, h[q], anyinf);
            }
        }
        for (; c < cb; ++c) { // the rest: odd chunk, padding columns, rows past N
            const int64_t col = c * 32 + 4 * tig;
            Chunk h;
            h.q00 = *reinterpret_cast<const uint2 *>(x0 + col * s0);
            h.q10 = *reinterpret_cast<const uint2 *>(x1 + col * s1);
            h.q01 = *reinterpret_cast<const uint2 *>(x0 + (col + 16) * s0);
            h.q11 = *reinterpret_cast<const uint2 *>(x1 + (col + 16) * s1);
            h.wf = wfrag[c * 32 + lane];
            if (c >= nfull) { // padding columns (+inf in X) read as 0
                auto m = [&](int64_t c0) -> uint2 {
                    return make_uint2((c0 < w ? 0xFFFFu : 0u) | (c0 + 1 < w ? 0xFFFF0000u : 0u),
                                      (c0 + 2 < w ? 0xFFFFu : 0u) | (c0 + 3 < w ? 0xFFFF0000u : 0u));
                };
                const uint2 ma = m(col), mb = m(col + 16);
                h.q00.x &= ma.x, h.q00.y &= ma.y, h.q10.x &= ma.x, h.q10.y &= ma.y;
                h.q01.x &= mb.x, h.q01.y &= mb.y, h.q11.x &= mb.x, h.q11.y &= mb.y;
            }
            mma_chunk<FIX>(acc, h, anyinf);
        }
        tile_hash(acc, tig, r0, r1, v0, v1, rw, rwm, hacc);
    }
    warp_flush<FIX>(hacc, anyinf, tcs);
}

// FIX (the +inf remapping) only where it can matter: the first power, and any power after one
// that held +inf (prev: the previous power's {H, flags}); a power of A(D_n) after an all-finite
// one is all-finite.  A power that holds +inf anyway is flagged void (k_stats_sym then hashes it).
__global__ void __launch_bounds__(256, MP_FPTC_MINB)
    k_fp_tc(const uint16_t *__restrict__ X, int64_t ld, int64_t N, int64_t w, const uint4 *__restrict__ wfrag,
            const uint64_t *__restrict__ rw, const uint64_t *__restrict__ rwm, int64_t ntiles, int64_t nparts,
            int64_t chunks_per_part, int64_t nchunks, unsigned long long *__restrict__ tcs,
            const unsigned long long *__restrict__ prev)
{
    __shared__ __align__(16) uint16_t zero_row[32];
    if (threadIdx.x < 32) zero_row[threadIdx.x] = 0;
    __syncthreads();
    if (!prev || prev[1] != 0)
        fp_tc_body<true>(X, ld, N, w, wfrag, rw, rwm, ntiles, nparts, chunks_per_part, nchunks, tcs, zero_row);
    else
        fp_tc_body<false>(X, ld, N, w, wfrag, rw, rwm, ntiles, nparts, chunks_per_part, nchunks, tcs, zero_row);
}

} // namespace

cudaError_t launch_fp_tc_weights(const int32_t *gcol, const int32_t *sigma, int64_t w, int64_t ld, uint4 *wfrag,
                                 cudaStream_t s)
{
    const int64_t nchunks = ld / 32;
    const int64_t g = std::max<int64_t>(1, std::min<int64_t>((nchunks * 32 + 255) / 256, 148 * 16));
    k_fp_tc_weights<<<(unsigned)g, 256, 0, s>>>(gcol, sigma, w, nchunks, wfrag);
    return cudaGetLastError();
}

cudaError_t launch_fp_tc(const uint16_t *X, int64_t ld, int64_t N, int64_t w, const uint4 *wfrag, const uint64_t *rw,
                         const uint64_t *rwm, unsigned long long *tcs, cudaStream_t s, const unsigned long long *prev)
{
    const int64_t nchunks = (w + 31) / 32, ntiles = (N + 15) / 16;
    // one wave of MP_FPTC_MINB x 8 resident warps per SM: split the columns only when the
    // 16-row tiles fill less than half of it
    const int64_t want = 148 * 8 * MP_FPTC_MINB;
    const int64_t nparts = std::max<int64_t>(1, std::min<int64_t>(nchunks, want / ntiles));
    const int64_t cpp = (nchunks + nparts - 1) / nparts;
    const int64_t warps = ntiles * nparts;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((warps + 7) / 8, 148 * MP_FPTC_MINB));
    k_fp_tc<<<grid, 256, 0, s>>>(X, ld, N, w, wfrag, rw, rwm, ntiles, nparts, cpp, nchunks, tcs, prev);
    return cudaGetLastError();
}

} // namespace mp
