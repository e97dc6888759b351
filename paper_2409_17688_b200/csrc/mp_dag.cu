// Row-inclusion reuse for the transfer matrix A(D_n) (DESIGN.md section 5 "Row-inclusion
// reuse").  Product code only; shares nothing with oracle/.
//
// Whether p can follow q depends on q only through its zero positions z(q) and its
// 2-positions t(q): rule (1) asks p_i = 0 wherever q_i = 2, rules (2)-(3) count q_i = 0 among
// the neighbours of p_i.  The label of the arc q -> p is the number of zeros of p, a
// function of p alone.  Let q' be q with ONE letter q_i in {0, 1} turned into a 2.  Every p that
// can follow q' has p_i = 0 (rule 1), so no rule applies at position i, and at every other
// position the rules read the same letters of q and q'; hence p can follow q, with the same
// label: row q' of A is row q restricted to a subset of its support.  For every power,
//     (A^k)_(q, j) = min( min over parents q' of (A^k)_(q', j),
//                         min over l in extra(q) of a_ql + (A^{k-1})_(l, j) ),
// extra(q) = supp(q) minus the union of the parents' supports -- the same minimum over the same
// terms (min is idempotent), regrouped.  The SpMM kernel runs on the extra entries only
// (about 3 % of nnz(A) for n >= 10) and a fold pass per level of the parent DAG (a parent has one
// more 2, so there are at most n + 1 levels) takes the minimum with the parents' finished rows.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "mp_internal.h"
#include "mp_kernels.h"

namespace mp {

namespace {

// Base-3 value of a word with letter 0 (the top row) most significant: the lexicographic order
// of A(D_n) (G5) is the order of these keys.
__device__ __forceinline__ uint32_t word_key(const WordMask &w, int n)
{
    uint32_t k = 0;
    for (int i = 0; i < n; ++i) k = 3 * k + ((w.o >> i) & 1u) + 2 * ((w.t >> i) & 1u);
    return k;
}

__global__ void k_word_keys(const WordMask *__restrict__ w, int64_t N, int n, uint32_t *__restrict__ keys)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
        keys[i] = word_key(w[i], n);
}

__device__ __forceinline__ int64_t find_key(const uint32_t *__restrict__ keys, int64_t N, uint32_t k)
{
    int64_t lo = 0, hi = N;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (keys[mid] < k) lo = mid + 1;
        else hi = mid;
    }
    return (lo < N && keys[lo] == k) ? lo : -1;
}

// parents of q: the words q with one letter 0 or 1 turned into a 2 that are correct words
// (count pass if pidx == nullptr, else fill from off[q])
__global__ void k_dag_parents(const WordMask *__restrict__ w, const uint32_t *__restrict__ keys, int64_t N, int n,
                              const int64_t *__restrict__ off, int32_t *__restrict__ cnt, int32_t *__restrict__ pidx)
{
    uint32_t pw3[16];
    pw3[0] = 1;
    for (int i = 1; i < 16; ++i) pw3[i] = 3 * pw3[i - 1];
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < N; q += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t kq = keys[q];
        int c = 0;
        int64_t o = pidx ? off[q] : 0;
        for (int b = 0; b < n; ++b) {
            if ((w[q].t >> b) & 1u) continue;
            const uint32_t up = ((w[q].o >> b) & 1u) ? 1u : 2u;         // letter b: 1 -> 2 or 0 -> 2
            const int64_t p = find_key(keys, N, kq + up * pw3[n - 1 - b]);
            if (p < 0) continue;
            if (pidx) pidx[o++] = (int32_t)p;
            ++c;
        }
        if (!pidx) cnt[q] = c;
    }
}

// level[q] = 0 without parents, else 1 + max level of the parents (one relaxation pass; n + 1
// passes reach the fixed point: a parent has one more 2)
__global__ void k_dag_level(const int64_t *__restrict__ off, const int32_t *__restrict__ pidx, int64_t N,
                            int32_t *__restrict__ level)
{
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < N; q += (int64_t)gridDim.x * blockDim.x) {
        int l = 0;
        for (int64_t e = off[q]; e < off[q + 1]; ++e) l = max(l, level[pidx[e]] + 1);
        level[q] = l;
    }
}

__global__ void k_level_hist(const int32_t *__restrict__ level, int64_t N, int32_t *__restrict__ hist)
{
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < N; q += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&hist[level[q]], 1);
}

// rows grouped by level (the order inside a level is irrelevant: a level's rows are folded
// independently); cursor[] zeroed by the caller
__global__ void k_level_scatter(const int32_t *__restrict__ level, int64_t N, const int64_t *__restrict__ lptr,
                                unsigned long long *__restrict__ cursor, int32_t *__restrict__ lrows)
{
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < N; q += (int64_t)gridDim.x * blockDim.x) {
        const int l = level[q];
        lrows[lptr[l] + (int64_t)atomicAdd(cursor + l, 1ull)] = (int32_t)q;
    }
}

// extra(q) = supp(q) minus the parents' supports, as bitsets (warp per row, lanes over words);
// *bad is set if some parent's support is not inside supp(q) (impossible for A(D_n), whose
// identity the run has verified; the check keeps a wrong structure from ever changing a result)
__global__ void k_extra_bits(const uint32_t *__restrict__ bits, int64_t nw, int64_t N, const int64_t *__restrict__ off,
                             const int32_t *__restrict__ pidx, uint32_t *__restrict__ ebits, int *__restrict__ bad)
{
    const int lane = threadIdx.x & 31;
    bool wrong = false;
    for (int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < N;
         q += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t e0 = off[q], e1 = off[q + 1];
        for (int64_t k = lane; k < nw; k += 32) {
            const uint32_t s = bits[q * nw + k];
            uint32_t m = s;
            for (int64_t e = e0; e < e1; ++e) {
                const uint32_t pb = bits[(int64_t)pidx[e] * nw + k];
                wrong |= (pb & ~s) != 0u;
                m &= ~pb;
            }
            ebits[q * nw + k] = m;
        }
    }
    if (wrong) atomicOr(bad, 1);
}

// (A^k)_(q, :) = min((A^k)_(q, :), (A^k)_(p, :)) over the parents p of the rows q of one level
// (the parents' rows are final: they belong to earlier levels).  A warp takes one row segment of
// kFoldSeg columns (32 B per lane, 4 x 16-byte loads per row read): lane e < #parents loads the
// e-th parent index once and shuffles it to the warp, so the row's metadata costs a few
// instructions per 1 KB of data.  Work items go segment-major (every row of the level for
// segment 0, then segment 1, ...), so the warps running at one time read the parents' rows of
// one segment column, which L2 then serves to the parents' other children.
#ifndef MP_FOLD_SEG
#define MP_FOLD_SEG 1024
#endif
#ifndef MP_FOLD_PAR
#define MP_FOLD_PAR 2
#endif
#ifndef MP_FOLD_MINB
#define MP_FOLD_MINB 4
#endif
constexpr int kFoldSeg = MP_FOLD_SEG; // columns per warp item (ld is a multiple of 64: the last is partial)
constexpr int kFoldQ = kFoldSeg / 256; // 16-byte loads per lane and row
constexpr int kFoldPar = MP_FOLD_PAR;  // parents loaded per step
__global__ void __launch_bounds__(256, MP_FOLD_MINB) k_fold(const int32_t *__restrict__ lrows, int64_t nrows,
                                              const int64_t *__restrict__ off, const int32_t *__restrict__ pidx,
                                              uint16_t *__restrict__ C, int64_t ldc)
{
    // launched as a programmatic dependent: the previous kernel's writes (the SpMM's rows, the
    // lower levels' folds) are complete and visible after this wait
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    const int lane = threadIdx.x & 31;
    const int64_t nseg = (ldc + kFoldSeg - 1) / kFoldSeg, items = nrows * nseg;
    for (int64_t it = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < items;
         it += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t seg = it / nrows, r = it - seg * nrows;
        const int64_t q = lrows[r];
        const int64_t e0 = off[q], np = off[q + 1] - e0;
        const int32_t mine = lane < np ? pidx[e0 + lane] : 0;
        uint16_t *row = C + q * ldc + seg * kFoldSeg;
        const int ncols = (int)(ldc - seg * kFoldSeg < kFoldSeg ? ldc - seg * kFoldSeg : kFoldSeg);
#if MP_DEBUG_CHECKS
        if (q < 0 || np > 32) __trap();
#endif
        uint4 v[kFoldQ];
#pragma unroll
        for (int h = 0; h < kFoldQ; ++h) {
            const int col = 256 * h + 8 * lane;
            v[h] = col < ncols ? *reinterpret_cast<const uint4 *>(row + col) : make_uint4(0, 0, 0, 0);
        }
        // parents kFoldPar at a time: kFoldPar x kFoldQ 16-byte loads per lane in flight (a
        // missing parent repeats the last one: min is idempotent)
        for (int e = 0; e < np; e += kFoldPar) {
            uint4 u[kFoldPar][kFoldQ];
#pragma unroll
            for (int j = 0; j < kFoldPar; ++j) {
                const int64_t pj = __shfl_sync(0xFFFFFFFFu, mine, e + j < np ? e + j : (int)np - 1);
#if MP_DEBUG_CHECKS
                if (pj < 0 || pj == q) __trap();
#endif
                const uint16_t *rj = C + pj * ldc + seg * kFoldSeg;
#pragma unroll
                for (int h = 0; h < kFoldQ; ++h) {
                    const int col = 256 * h + 8 * lane;
                    u[j][h] = col < ncols ? __ldcg(reinterpret_cast<const uint4 *>(rj + col)) : make_uint4(0, 0, 0, 0);
                }
            }
#pragma unroll
            for (int j = 0; j < kFoldPar; ++j)
#pragma unroll
                for (int h = 0; h < kFoldQ; ++h) {
                    v[h].x = __vminu2(v[h].x, u[j][h].x);
                    v[h].y = __vminu2(v[h].y, u[j][h].y);
                    v[h].z = __vminu2(v[h].z, u[j][h].z);
                    v[h].w = __vminu2(v[h].w, u[j][h].w);
                }
        }
#pragma unroll
        for (int h = 0; h < kFoldQ; ++h) {
            const int col = 256 * h + 8 * lane;
            if (col < ncols) *reinterpret_cast<uint4 *>(row + col) = v[h];
        }
    }
}

int grid_rows(int64_t work, int per_block)
{
    const int64_t g = (work + per_block - 1) / per_block;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16));
}

} // namespace

cudaError_t build_row_dag(const WordMask *words, int64_t N, int n, RowDag &d, cudaStream_t s,
                          cudaError_t (*alloc)(void **, size_t, void *), void *actx, int64_t *launches)
{
    cudaError_t e;
    auto A = [&](auto *&p, size_t bytes) { return alloc((void **)&p, std::max<size_t>(bytes, 16), actx); };
    uint32_t *keys = nullptr;
    int32_t *cnt = nullptr, *hist = nullptr;
    if ((e = A(keys, (size_t)N * 4)) != cudaSuccess) return e;
    if ((e = A(cnt, (size_t)N * 4)) != cudaSuccess) return e;
    if ((e = A(d.off, (size_t)(N + 1) * 8)) != cudaSuccess) return e;
    if ((e = A(d.level, (size_t)N * 4)) != cudaSuccess) return e;
    if ((e = A(d.lrows, (size_t)N * 4)) != cudaSuccess) return e;
    if ((e = A(hist, 32 * 8)) != cudaSuccess) return e;
    if ((e = A(d.lptr_dev, 33 * 8)) != cudaSuccess) return e;
    if ((e = A(d.bad, 16)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(d.bad, 0, sizeof(int), s)) != cudaSuccess) return e;
    const int gb = grid_rows(N, 256);
    k_word_keys<<<gb, 256, 0, s>>>(words, N, n, keys);
    k_dag_parents<<<gb, 256, 0, s>>>(words, keys, N, n, nullptr, cnt, nullptr);
    *launches += 2;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // offsets on the host (N <= 131562 counts): one copy each way
    std::vector<int32_t> hc((size_t)N);
    if ((e = cudaMemcpyAsync(hc.data(), cnt, (size_t)N * 4, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    std::vector<int64_t> ho((size_t)N + 1, 0);
    for (int64_t q = 0; q < N; ++q) ho[(size_t)q + 1] = ho[(size_t)q] + hc[(size_t)q];
    d.parents = ho[(size_t)N];
    if ((e = A(d.idx, (size_t)d.parents * 4)) != cudaSuccess) return e;
    if ((e = cudaMemcpyAsync(d.off, ho.data(), ho.size() * 8, cudaMemcpyHostToDevice, s)) != cudaSuccess) return e;
    k_dag_parents<<<gb, 256, 0, s>>>(words, keys, N, n, d.off, nullptr, d.idx);
    if ((e = cudaMemsetAsync(d.level, 0, (size_t)N * 4, s)) != cudaSuccess) return e;
    for (int pass = 0; pass <= n; ++pass) k_dag_level<<<gb, 256, 0, s>>>(d.off, d.idx, N, d.level);
    if ((e = cudaMemsetAsync(hist, 0, 32 * 4, s)) != cudaSuccess) return e;
    k_level_hist<<<gb, 256, 0, s>>>(d.level, N, hist);
    *launches += (int64_t)n + 3;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    int32_t hh[32];
    if ((e = cudaMemcpyAsync(hh, hist, sizeof(hh), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    d.levels = 0;
    d.lptr.assign(1, 0);
    for (int l = 0; l < 32 && hh[l] > 0; ++l) {
        d.lptr.push_back(d.lptr.back() + hh[l]);
        d.levels = l + 1;
    }
    if (d.lptr.back() != N) return cudaErrorUnknown; // levels are contiguous from 0
    if ((e = cudaMemcpyAsync(d.lptr_dev, d.lptr.data(), d.lptr.size() * 8, cudaMemcpyHostToDevice, s)) != cudaSuccess)
        return e;
    // the level lists in a fixed order (MP_FOLD_ORDER: q = ascending row, the default; p = by
    // first parent, then row; s = the order of the device scatter's atomics)
    const char *fo = getenv("MP_FOLD_ORDER");
    const char order = fo && (fo[0] == 'p' || fo[0] == 's') ? fo[0] : 'q';
    std::vector<int32_t> hl;
    {   // fold_rows = sum over levels >= 1 of (2 x rows + distinct parents): levels and parent
        // lists to the host once per DAG (N + #parents ints)
        std::vector<int32_t> lv((size_t)N), pi((size_t)std::max<int64_t>(d.parents, 1));
        if ((e = cudaMemcpyAsync(lv.data(), d.level, (size_t)N * 4, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
        if (d.parents > 0 &&
            (e = cudaMemcpyAsync(pi.data(), d.idx, (size_t)d.parents * 4, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
            return e;
        if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
        std::vector<std::vector<int32_t>> by((size_t)d.levels);
        for (int64_t q = 0; q < N; ++q) by[(size_t)lv[(size_t)q]].push_back((int32_t)q);
        std::vector<int32_t> seen((size_t)N, -1);
        d.fold_rows = 0;
        for (int l = 1; l < d.levels; ++l)
            for (const int32_t q : by[(size_t)l]) {
                d.fold_rows += 2;
                for (int64_t k = ho[(size_t)q]; k < ho[(size_t)q + 1]; ++k)
                    if (seen[(size_t)pi[(size_t)k]] != l) {
                        seen[(size_t)pi[(size_t)k]] = l;
                        ++d.fold_rows;
                    }
            }
        if (order != 's') {
            hl.reserve((size_t)N);
            for (auto &rows : by) {
                if (order == 'p')
                    std::stable_sort(rows.begin(), rows.end(), [&](int32_t a, int32_t b) {
                        const int32_t pa = ho[(size_t)a] < ho[(size_t)a + 1] ? pi[(size_t)ho[(size_t)a]] : -1;
                        const int32_t pb = ho[(size_t)b] < ho[(size_t)b + 1] ? pi[(size_t)ho[(size_t)b]] : -1;
                        return pa < pb;
                    });
                hl.insert(hl.end(), rows.begin(), rows.end());
            }
        }
    }
    if (order != 's') {
        if ((e = cudaMemcpyAsync(d.lrows, hl.data(), (size_t)N * 4, cudaMemcpyHostToDevice, s)) != cudaSuccess) return e;
    } else {
        if ((e = cudaMemsetAsync(hist, 0, 32 * 8, s)) != cudaSuccess) return e; // reused as the cursors
        k_level_scatter<<<gb, 256, 0, s>>>(d.level, N, d.lptr_dev, reinterpret_cast<unsigned long long *>(hist),
                                           d.lrows);
        *launches += 1;
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    return cudaStreamSynchronize(s); // d.lptr (host) and ho go out of scope safely
}

cudaError_t launch_extra_bits(const uint32_t *bits, int64_t nw, int64_t N, const RowDag &d, uint32_t *ebits,
                              cudaStream_t s)
{
    k_extra_bits<<<grid_rows(N * 32, 256), 256, 0, s>>>(bits, nw, N, d.off, d.idx, ebits, d.bad);
    return cudaGetLastError();
}

static bool fold_pdl()
{
    const char *e = getenv("MP_FOLD_PDL"); // read per call: experiments switch it
    return !(e && e[0] == '0');
}

cudaError_t launch_folds(const RowDag &d, uint16_t *C, int64_t ldc, int64_t ncols, cudaStream_t s, int *launches)
{
    for (int l = 1; l < d.levels; ++l) {
        const int64_t nr = d.lptr[(size_t)l + 1] - d.lptr[(size_t)l];
        const int64_t items = nr * ((ncols + kFoldSeg - 1) / kFoldSeg);
        // a grid of at most 148 x 8 blocks of 8 warps: the running warps are a contiguous range
        // of items (the segment-major order above relies on it)
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((items + 7) / 8, 148 * 8));
        // programmatic dependent launch: this level's grid is set up while the previous kernel
        // (the SpMM or the level before) drains; k_fold waits for that kernel's completion
        // (griddepcontrol.wait) before its first load.  MP_FOLD_PDL=0: plain launches.
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)grid);
        cfg.blockDim = dim3(256);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = fold_pdl() ? 1 : 0;
        const cudaError_t le = cudaLaunchKernelEx(&cfg, k_fold, (const int32_t *)(d.lrows + d.lptr[(size_t)l]), nr,
                                                  (const int64_t *)d.off, (const int32_t *)d.idx, C, ldc);
        if (le != cudaSuccess) return le;
        if (launches) ++*launches;
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

} // namespace mp
