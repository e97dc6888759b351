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
// chunks, loads its 4 x 4 u16 of X per chunk, maps +inf to 0xFFFF, splits the bytes with PRMT
// and issues 4 MMAs (2 planes x {b, b'}).  The kernel is bound by reading X once; the issue
// work per entry is about 0.1 instruction (the CUDA-core k_stats_sym needed about 20).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "mp_internal.h"
#include "mp_kernels.h"

namespace mp {

namespace {

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

// +inf (0x7FFF) -> 0xFFFF in both halves; counts the +inf halves into *cnt
__device__ __forceinline__ uint32_t fix_inf(uint32_t v, uint32_t valid, int &cnt)
{
    const uint32_t m = __vcmpeq2(v, 0x7FFF7FFFu) & valid; // 0xFFFF per +inf half
    cnt += __popc(m) >> 4;
    return (v | m) & valid;
}

// Work item = (16-row tile, column part): the part's chunks [c0, c1).
__global__ void __launch_bounds__(256)
    k_fp_tc(const uint16_t *__restrict__ X, int64_t ld, int64_t N, int64_t w, const uint4 *__restrict__ wfrag,
            const uint64_t *__restrict__ rw, const uint64_t *__restrict__ rwm, int64_t ntiles, int64_t nparts,
            int64_t chunks_per_part, int64_t nchunks, unsigned long long *__restrict__ tcs)
{
    const int lane = threadIdx.x & 31, n = lane >> 2, tig = lane & 3;
    unsigned long long hacc = 0;
    int infc = 0;
    const int64_t items = ntiles * nparts;
    for (int64_t it = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < items;
         it += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t tile = it / nparts, part = it - tile * nparts;
        const int64_t r0 = tile * 16 + n, r1 = r0 + 8; // this lane's two rows
        const bool v0 = r0 < N, v1 = r1 < N;
        const int64_t ca = part * chunks_per_part, cb = min(nchunks, ca + chunks_per_part);
        int acc[4][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}, {0, 0, 0, 0}, {0, 0, 0, 0}}; // {p0 b, p0 b', p1 b, p1 b'}
        const uint16_t *x0 = X + (v0 ? r0 : 0) * ld, *x1 = X + (v1 ? r1 : 0) * ld;
        for (int64_t c = ca; c < cb; ++c) {
            const int64_t col = c * 32 + 4 * tig;
            const uint2 q00 = *reinterpret_cast<const uint2 *>(x0 + col);      // row r0, cols +0..3
            const uint2 q10 = *reinterpret_cast<const uint2 *>(x1 + col);      // row r1
            const uint2 q01 = *reinterpret_cast<const uint2 *>(x0 + col + 16); // row r0, cols +16..19
            const uint2 q11 = *reinterpret_cast<const uint2 *>(x1 + col + 16);
            const uint4 wf = wfrag[c * 32 + lane];
            // validity masks per u16 half: rows < N, columns < w
            auto vm = [&](bool rowok, int64_t c0) -> uint2 {
                uint32_t m0 = 0, m1 = 0;
                if (rowok) {
                    m0 = (c0 < w ? 0xFFFFu : 0u) | (c0 + 1 < w ? 0xFFFF0000u : 0u);
                    m1 = (c0 + 2 < w ? 0xFFFFu : 0u) | (c0 + 3 < w ? 0xFFFF0000u : 0u);
                }
                return make_uint2(m0, m1);
            };
            const uint2 m00 = vm(v0, col), m10 = vm(v1, col), m01 = vm(v0, col + 16), m11 = vm(v1, col + 16);
            const uint32_t y00x = fix_inf(q00.x, m00.x, infc), y00y = fix_inf(q00.y, m00.y, infc);
            const uint32_t y10x = fix_inf(q10.x, m10.x, infc), y10y = fix_inf(q10.y, m10.y, infc);
            const uint32_t y01x = fix_inf(q01.x, m01.x, infc), y01y = fix_inf(q01.y, m01.y, infc);
            const uint32_t y11x = fix_inf(q11.x, m11.x, infc), y11y = fix_inf(q11.y, m11.y, infc);
            // A fragments: a0 = (row n, cols 4 tig..), a1 = (row n + 8, ..), a2 / a3 = cols + 16
            const uint32_t lo[4] = {__byte_perm(y00x, y00y, 0x6420), __byte_perm(y10x, y10y, 0x6420),
                                    __byte_perm(y01x, y01y, 0x6420), __byte_perm(y11x, y11y, 0x6420)};
            const uint32_t hi[4] = {__byte_perm(y00x, y00y, 0x7531), __byte_perm(y10x, y10y, 0x7531),
                                    __byte_perm(y01x, y01y, 0x7531), __byte_perm(y11x, y11y, 0x7531)};
            imma(acc[0], lo, wf.x, wf.y);
            imma(acc[1], lo, wf.z, wf.w);
            imma(acc[2], hi, wf.x, wf.y);
            imma(acc[3], hi, wf.z, wf.w);
        }
        // D fragment: d0, d1 = (row n, bytes 2 tig, 2 tig + 1), d2, d3 = (row n + 8, same bytes).
        // u = sum_{p, t} 256^(p + t) D_p[t] over this lane's two bytes, then over the group's
        // four lanes (all eight bytes): sums of 32-bit values as unsigned, mod 2^64.
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
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        hacc += __shfl_xor_sync(0xFFFFFFFFu, hacc, o);
        infc += __shfl_xor_sync(0xFFFFFFFFu, infc, o);
    }
    if (lane == 0) {
        if (hacc) atomicAdd(tcs + 0, hacc);
        if (infc) atomicAdd(tcs + 1, (unsigned long long)infc);
    }
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
                         const uint64_t *rwm, unsigned long long *tcs, cudaStream_t s)
{
    const int64_t nchunks = (w + 31) / 32, ntiles = (N + 15) / 16;
    // about 16 warps per SM: split the columns when there are too few 16-row tiles
    const int64_t want = 148 * 16;
    const int64_t nparts = std::max<int64_t>(1, std::min<int64_t>(nchunks, (want + ntiles - 1) / ntiles));
    const int64_t cpp = (nchunks + nparts - 1) / nparts;
    const int64_t warps = ntiles * nparts;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((warps + 7) / 8, 148 * 8));
    k_fp_tc<<<grid, 256, 0, s>>>(X, ld, N, w, wfrag, rw, rwm, ntiles, nparts, cpp, nchunks, tcs);
    return cudaGetLastError();
}

} // namespace mp
