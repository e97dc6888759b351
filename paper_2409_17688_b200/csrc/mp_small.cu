// Small-N latency path (N <= 256, e.g. A(D_n) for n <= 6): the WHOLE power-until-periodic run
// -- every product A^k = A (x) A^{k-1} (Algorithm 2), its statistics (a4), the
// first-repeat search with its exact compare (a5; Lemma 1) -- in ONE launch of one
// thread-block cluster, with one host read of the result at the end.
// "Small-N path".  Product code only; shares nothing with oracle/.
//
// CTA c of the cluster owns the 64 columns [64c, 64c + 64) of every power (a lane holds two of
// them as a packed u16 pair).  Column j of A^k depends only on column j of A^{k-1} (left
// multiplication by the fixed A, G8), so the CTAs never exchange matrix data: A's finite entries
// (row lists) and the CTA's column block of A^{k-1} and A^k live in shared memory, and only the
// per-power statistics (fingerprint, +inf count, diagonal minimum, first finite entry) and the
// exact-compare mismatch counts cross the cluster, through distributed shared memory.  Every
// power's column block is also written to a history buffer in global memory (L2-resident:
// at most 64 x 256 x 256 x 2 B) for the exact compares against earlier powers.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "mp_internal.h"
#include "mp_kernels.h"

namespace cg = cooperative_groups;

namespace mp {

namespace {

__device__ __forceinline__ uint32_t lds32(uint32_t addr)
{
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(v) : "r"(addr));
    return v;
}

constexpr int kSmThreads = 512; // at most 16 warps; warp w computes rows w, w + nwarps, ...
constexpr int kSmWarps = kSmThreads / 32;

struct Stats { // the per-power statistics of k_stats (mp_power_stats), int64 fields
    unsigned long long fp, inf;
    long long dmin, ref;
};

__device__ __forceinline__ unsigned long long shfl_xor_u64(unsigned long long v, int m)
{
    const unsigned lo = __shfl_xor_sync(0xFFFFFFFFu, (unsigned)v, m);
    const unsigned hi = __shfl_xor_sync(0xFFFFFFFFu, (unsigned)(v >> 32), m);
    return ((unsigned long long)hi << 32) | lo;
}

// Butterfly reduction of the statistics over the first `width` lanes (a power of two): the
// fingerprint as 64 bits, the +inf count, diagonal minimum and first-finite key as 32 bits
// (N <= 256: t = i N + j < 2^16, so a key (t << 16) | x < 2^32; no key = 0x7FFF..F maps to
// 0xFFFFFFFF and back).
__device__ __forceinline__ void reduce_stats(Stats &s, int width)
{
    // whole-warp reductions (redux.sync); lanes outside `width` hold the identity, so the
    // result is the same.  The 64-bit sum in 16/16/32-bit limbs: at most 32 terms, no limb sum
    // overflows except the top one, which is taken mod 2^32 as the sum is mod 2^64.
    (void)width;
    const uint32_t inf = __reduce_add_sync(0xFFFFFFFFu, (uint32_t)s.inf);
    const uint32_t dmin = __reduce_min_sync(0xFFFFFFFFu, (uint32_t)s.dmin);
    const uint32_t ref =
        __reduce_min_sync(0xFFFFFFFFu, s.ref == 0x7FFFFFFFFFFFFFFFll ? 0xFFFFFFFFu : (uint32_t)s.ref);
    const uint32_t l0 = __reduce_add_sync(0xFFFFFFFFu, (uint32_t)(s.fp & 0xFFFFu));
    const uint32_t l1 = __reduce_add_sync(0xFFFFFFFFu, (uint32_t)((s.fp >> 16) & 0xFFFFu));
    const uint32_t hi = __reduce_add_sync(0xFFFFFFFFu, (uint32_t)(s.fp >> 32));
    s.fp = ((unsigned long long)hi << 32) + ((unsigned long long)l1 << 16) + (unsigned long long)l0;
    s.inf = inf;
    s.dmin = dmin;
    s.ref = ref == 0xFFFFFFFFu ? 0x7FFFFFFFFFFFFFFFll : (long long)ref;
}

// Candidate test of the forward first-repeat search (the rule of mp_repeat_candidate in
// mp_api.cu, restated for the device).
__device__ bool candidate(const Stats &k, const Stats &j, unsigned long long S, int *c)
{
    if (k.inf != j.inf) return false;
    const long long kInfRef = 0x7FFFFFFFFFFFFFFFll;
    const bool ak = k.ref == kInfRef, aj = j.ref == kInfRef;
    if (ak || aj) {
        *c = 0;
        return ak == aj;
    }
    if ((k.ref >> 16) != (j.ref >> 16)) return false;
    *c = (int)(k.ref & 0xFFFF) - (int)(j.ref & 0xFFFF);
    if (k.inf > 0) return true; // +inf present: the exact compare decides
    return k.fp - j.fp == (unsigned long long)(long long)*c * S;
}

} // namespace

// Cluster layout: C = ceil(N / 64) column blocks x R row parts (small_run_shape); CTA (c, r)
// (cluster rank c + C r) computes rows [r0, r1) of column block c of every power and writes
// them into its own and its R - 1 row peers' copies of that column block (distributed shared
// memory), so each CTA holds the whole block of A^k for the next product.
// sigma (may be null): a symmetry hint to verify (every finite A_il must reappear at
// (sigma i, sigma l)); the run itself computes every column.
// out[]: status (0 ok, 1 symmetry hint violated, 2 range, 4 not periodic, -1 too many entries
// for shared memory), mu, lambda, offset, k_last, dense_from, then diag_min[k] and
// fingerprint[k] for k = 0..max_k.
__global__ void __launch_bounds__(kSmThreads, 1)
    k_small_run(const uint16_t *__restrict__ A, int64_t lda, int N, int C, int max_k, int max_nnz,
                const int32_t *__restrict__ sigma, uint16_t *__restrict__ hist, unsigned long long S,
                long long *__restrict__ out)
{
    extern __shared__ __align__(16) uint8_t smem[];
    cg::cluster_group cluster = cg::this_cluster();
    const int nct = (int)cluster.num_blocks(), rk = (int)cluster.block_rank();
    const int R = nct / C, c = rk % C, r = rk / C;
    // a cluster of one CTA needs only the block barrier
    auto csync = [&]() {
        if (nct > 1) cluster.sync();
        else __syncthreads();
    };
    const int rows_per = (N + R - 1) / R;
    const int r0 = min(N, r * rows_per), r1 = min(N, r0 + rows_per), nr = r1 - r0;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nthreads = blockDim.x, nwarps = nthreads >> 5; // fewer warps for few rows
    const int ldh = 64 * C;               // history pitch (columns of all CTAs)
    const int64_t hsz = (int64_t)N * ldh; // one power in the history

    // shared memory: X blocks (2 x N x 32 u32) | row weights of the own rows | row pointers |
    // entries of the own rows | statistics history | per-warp partials | cluster exchange (2
    // parity buffers) | mismatch exchange | flags
    uint32_t *Xa = reinterpret_cast<uint32_t *>(smem);
    uint32_t *Xb = Xa + N * 32;
    uint64_t *rw = reinterpret_cast<uint64_t *>(Xb + N * 32); // [rows_per] s(2i)
    int32_t *rptr = reinterpret_cast<int32_t *>(rw + rows_per);
    // entry e of an own row: {byte offset of X row l in a 32 x u32 block, a_il in both halves}
    uint2 *ent = reinterpret_cast<uint2 *>(rptr + ((rows_per + 4) & ~3));
    Stats *hs = reinterpret_cast<Stats *>(ent + ((max_nnz + 1) & ~1)); // [max_k + 1]
    Stats *wred = hs + (max_k + 1);                                       // [kSmWarps]
    Stats *xch = wred + kSmWarps;                                         // [2]: this CTA's partials
    long long *xmis = reinterpret_cast<long long *>(xch + 2);             // [2]: mismatch partials
    int *flags = reinterpret_cast<int *>(xmis + 2); // [0] range, [1] nnz, [2] candidate j, [3] c, [4] asym,
                                                    // [5] dense_from (at the end)

    const int j0 = 64 * c + 2 * lane, j1 = j0 + 1; // this lane's global columns
    const bool v0 = j0 < N, v1 = j1 < N;
    const uint64_t cw0 = v0 ? mix64(2 * (uint64_t)j0 + 1) : 0, cw1 = v1 ? mix64(2 * (uint64_t)j1 + 1) : 0;

    // ---- a2: row lists of the own rows, range and symmetry checks, X_1 block (every row).
    // A is read once with independent loads by every thread: the own rows into As (staged in
    // the Xb buffer: nr <= 64 rows of N u16 fit in N x 128 bytes) and the CTA's column block of
    // every row straight into Xa (X_1 in the device encoding); the passes below read shared memory.
    long long t_start = clock64();
    uint16_t *As = reinterpret_cast<uint16_t *>(Xb); // [nr][N]
    if (tid == 0) flags[0] = flags[1] = flags[4] = 0;
    for (int t = tid; t < nr; t += nthreads) rw[t] = mix64(2 * (uint64_t)(r0 + t));
    for (int t = tid; t < nr * N; t += nthreads) {
        const int ii = t / N, l = t - ii * N;
        As[t] = A[(int64_t)(r0 + ii) * lda + l];
    }
    for (int t = tid; t < N * 32; t += nthreads) { // X_1 = A[:, block], packed pairs
        const int i = t >> 5, ln = t & 31, ja = 64 * c + 2 * ln;
        const uint16_t a0 = ja < N ? A[(int64_t)i * lda + ja] : (uint16_t)kBndInf;
        const uint16_t a1 = ja + 1 < N ? A[(int64_t)i * lda + ja + 1] : (uint16_t)kBndInf;
        Xa[t] = (uint32_t)(a0 == kBndInf ? kDevInf : a0) | ((uint32_t)(a1 == kBndInf ? kDevInf : a1) << 16);
    }
    __syncthreads();
    for (int ii = warp; ii < nr; ii += nwarps) {
        const int i = r0 + ii;
        int cnt = 0;
        bool bad = false, asym = false;
        for (int l0 = 0; l0 < N; l0 += 32) {
            const int l = l0 + lane;
            const uint16_t x = l < N ? As[ii * N + l] : (uint16_t)kBndInf;
            bad |= x != kBndInf && x > kFiniteMax;
            if (sigma && x != kBndInf) asym |= A[(int64_t)sigma[i] * lda + sigma[l]] != x;
            cnt += __popc(__ballot_sync(0xFFFFFFFFu, x != kBndInf));
        }
        if (__any_sync(0xFFFFFFFFu, bad) && lane == 0) flags[0] = 1;
        if (__any_sync(0xFFFFFFFFu, asym) && lane == 0) flags[4] = 1;
        if (lane == 0) rptr[ii + 1] = cnt;
    }
    __syncthreads();
    if (tid == 0) {
        rptr[0] = 0;
        for (int ii = 0; ii < nr; ++ii) rptr[ii + 1] += rptr[ii];
        flags[1] = rptr[nr] > max_nnz;
    }
    csync(); // every CTA's flags are final: one decision for the whole cluster
    bool stop = false;
    int status = 0;
    for (int q = 0; q < nct; ++q) {
        const int *f = cluster.map_shared_rank(flags, q);
        if (f[0]) status = 2;
        else if (f[4] && status != 2) status = 1;
        else if (f[1] && status == 0) status = -1;
    }
    stop = status != 0;
    csync(); // nobody changes its flags before every CTA has read them
    if (stop) {
        if (rk == 0 && tid == 0) out[0] = status;
        return;
    }
    for (int ii = warp; ii < nr; ii += nwarps) {
        int e = rptr[ii];
        for (int l0 = 0; l0 < N; l0 += 32) {
            const int l = l0 + lane;
            const uint16_t x = l < N ? As[ii * N + l] : (uint16_t)kBndInf;
            const unsigned m = __ballot_sync(0xFFFFFFFFu, x != kBndInf);
            if (x != kBndInf) ent[e + __popc(m & ((1u << lane) - 1))] = make_uint2((uint32_t)l * 128u, (uint32_t)x * 0x10001u);
            e += __popc(m);
        }
    }
    __syncthreads(); // As (in Xb) is free again: A^2 goes there
    // MP_SMALL_PROFILE builds: clock64 phase sums of CTA 0 thread 0 (setup, product + statistics,
    // reductions + barrier, search) appended to out[] for the host to print
    long long t_setup = t_start, t_prod = 0, t_red = 0, t_search = 0, t_mark = t_setup;
    uint32_t *Xp = Xa, *Xc = Xb; // X_{k-1}, X_k (X_1 is in Xa)
    int xi = 0;                  // cluster exchange count (parity buffer)
    int mu = 0, lam = 0, off = 0, k_last = 0, dense_from = 0;
    bool found = false;
    int k = 1;
    const uint32_t xlane = (uint32_t)__cvta_generic_to_shared(Xa) + 4 * lane; // this lane's column pair
    t_setup = clock64() - t_setup;
    for (;; ++k) {
        t_mark = clock64();
        uint32_t *X = (k == 1) ? Xa : Xc;
        const uint32_t xp_s = xlane + (uint32_t)((Xp - Xa) * 4);
        // ---- A^k = A (x) A^{k-1} on the own rows of this block (k >= 2) with the a4
        // statistics: warp per row, lane per column pair, entries walked four at a time into
        // independent chains; each new row also goes to the R - 1 row peers.
        Stats st{0ull, 0ull, 0xFFFFll, 0x7FFFFFFFFFFFFFFFll};
        for (int ii = warp; ii < nr; ii += nwarps) {
            const int i = r0 + ii;
            uint32_t p;
            if (k >= 2) {
                uint32_t acc0 = 0xFFFFFFFFu, acc1 = 0xFFFFFFFFu, acc2 = 0xFFFFFFFFu, acc3 = 0xFFFFFFFFu;
                const int e0 = rptr[ii], e1 = rptr[ii + 1];
#if MP_DEBUG_CHECKS
                if (e0 < 0 || e1 < e0 || e1 > max_nnz) __trap();
                for (int q = e0; q < e1; ++q)
                    if (ent[q].x >= (uint32_t)N * 128u) __trap();
#endif
                int e = e0;
                for (; e + 4 <= e1; e += 4) {
                    const uint2 q0 = ent[e], q1 = ent[e + 1], q2 = ent[e + 2], q3 = ent[e + 3];
                    acc0 = __viaddmin_u16x2(q0.y, lds32(xp_s + q0.x), acc0);
                    acc1 = __viaddmin_u16x2(q1.y, lds32(xp_s + q1.x), acc1);
                    acc2 = __viaddmin_u16x2(q2.y, lds32(xp_s + q2.x), acc2);
                    acc3 = __viaddmin_u16x2(q3.y, lds32(xp_s + q3.x), acc3);
                }
                for (; e < e1; ++e) {
                    const uint2 q0 = ent[e];
                    acc0 = __viaddmin_u16x2(q0.y, lds32(xp_s + q0.x), acc0);
                }
                p = __vminu2(__vminu2(__vminu2(acc0, acc1), __vminu2(acc2, acc3)), 0x7FFF7FFFu); // G6 clamp
                X[i * 32 + lane] = p;
                for (int rr = 0; rr < R; ++rr) // the row peers' copies of this column block
                    if (rr != r) cluster.map_shared_rank(X, c + C * rr)[i * 32 + lane] = p;
            } else {
                p = X[i * 32 + lane];
            }
            // a4: fingerprint, +inf count, diagonal minimum, first finite entry (boundary
            // encoding 0xFFFF for +inf in the hash)
            const uint32_t x0 = p & 0xFFFFu, x1 = p >> 16;
            const uint64_t b0 = x0 >= kDevInf ? kBndInf : x0, b1 = x1 >= kDevInf ? kBndInf : x1;
            st.fp += rw[ii] * (cw0 * b0 + cw1 * b1);
            st.inf += (v0 && x0 >= kDevInf) + (v1 && x1 >= kDevInf);
            if (v0 && j0 == i) st.dmin = min(st.dmin, (long long)b0);
            if (v1 && j1 == i) st.dmin = min(st.dmin, (long long)b1);
            if (v0 && x0 < kDevInf) st.ref = min(st.ref, (((long long)i * N + j0) << 16) | (long long)x0);
            if (v1 && x1 < kDevInf) st.ref = min(st.ref, (((long long)i * N + j1) << 16) | (long long)x1);
        }
        reduce_stats(st, 32);
        if (lane == 0) wred[warp] = st;
        __syncthreads();
        if (warp == 0) { // the CTA's partial: lanes < 16 hold the warps' partials
            Stats s = lane < nwarps ? wred[lane] : Stats{0ull, 0ull, 0xFFFFll, 0x7FFFFFFFFFFFFFFFll};
            reduce_stats(s, kSmWarps); // lanes >= nwarps hold the identity
            if (nct == 1) { // a single CTA: its partial is the power's statistics
                if (lane == 0) hs[k] = s;
                if (!dense_from && s.inf == 0) dense_from = k;
                __syncwarp(); // hs[k] visible to warp 0's lanes (the search)
            } else if (lane == 0) {
                xch[xi & 1] = s;
            }
        }
        {
            const long long t = clock64();
            t_prod += t - t_mark;
            t_mark = t;
        }
        if (nct > 1) {
            csync(); // partials and the peers' rows of A^k visible cluster-wide
            if (warp == 0) { // lane q < nct reads CTA q's partial; every lane ends with the sum
                Stats g = lane < nct ? cluster.map_shared_rank(xch, lane)[xi & 1]
                                     : Stats{0ull, 0ull, 0xFFFFll, 0x7FFFFFFFFFFFFFFFll};
                reduce_stats(g, 16); // a cluster has at most 16 CTAs
                if (lane == 0) hs[k] = g;
                if (!dense_from && g.inf == 0) dense_from = k;
            }
            ++xi;
            __syncthreads();
        }
        // (one CTA: only warp 0 reads hs[], in the search below; the other warps' rows of A^k
        // are published by the search's barrier before anyone reads them)
        // the own rows of A^k go to the history after the barrier: the stores complete while the
        // next product runs (exact compares of later powers read them, ordered by the barriers
        // in between)
        for (int t = tid; t < nr * 32; t += nthreads)
            reinterpret_cast<uint32_t *>(hist + (int64_t)k * hsz + (int64_t)(r0 + (t >> 5)) * ldh + 64 * c)[t & 31] =
                X[r0 * 32 + t];
        {
            const long long t = clock64();
            t_red += t - t_mark;
            t_mark = t;
        }
        // ---- a5: forward first-repeat search, j = k-1 down to 1 (identical in every CTA)
        int jn = k - 1;
        while (!found) {
            if (warp == 0) { // lane t tests j = jn - t (32 at a time, descending): the highest hit
                const Stats sk = hs[k];
                int j = 0, cc = 0;
                for (int top = jn; top >= 1; top -= 32) {
                    const int jj = top - lane;
                    int c1 = 0;
                    const bool hit = jj >= 1 && candidate(sk, hs[jj], S, &c1);
                    const unsigned m = __ballot_sync(0xFFFFFFFFu, hit);
                    if (m) {
                        const int src = __ffs(m) - 1; // the lowest lane = the highest j
                        j = __shfl_sync(0xFFFFFFFFu, jj, src);
                        cc = __shfl_sync(0xFFFFFFFFu, c1, src);
                        break;
                    }
                }
                if (lane == 0) {
                    flags[2] = j;
                    flags[3] = cc;
                }
            }
            __syncthreads();
            const int j = flags[2], cc = flags[3];
            if (j < 1) break;
            // exact compare of the own rows: equal +inf pattern, X_k - X_j = cc on finite entries
            long long bad = 0;
            const uint16_t *Z = hist + (int64_t)j * hsz + 64 * c;
            for (int t = tid; t < nr * 32; t += nthreads) {
                const int i = r0 + (t >> 5);
                const uint32_t y = X[i * 32 + (t & 31)];
                const uint32_t z = reinterpret_cast<const uint32_t *>(Z + (int64_t)i * ldh)[t & 31];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (!(h ? v1 : v0)) continue;
                    const int yy = (int)((y >> (16 * h)) & 0xFFFFu), zz = (int)((z >> (16 * h)) & 0xFFFFu);
                    const bool yi = yy >= kDevInf, zi = zz >= kDevInf;
                    bad += (yi != zi) || (!yi && yy - zz != cc);
                }
            }
            for (int m = 16; m; m >>= 1) bad += (long long)shfl_xor_u64((unsigned long long)bad, m);
            if (lane == 0) wred[warp].fp = (unsigned long long)bad;
            __syncthreads();
            if (warp == 0) {
                long long b = lane < nwarps ? (long long)wred[lane].fp : 0;
                for (int m = 16; m; m >>= 1) b += (long long)shfl_xor_u64((unsigned long long)b, m);
                if (lane == 0) xmis[xi & 1] = b;
            }
            csync();
            long long total = 0;
            for (int q = 0; q < nct; ++q) total += cluster.map_shared_rank(xmis, q)[xi & 1];
            ++xi;
            if (total == 0) {
                found = true;
                mu = j;
                lam = k - j;
                off = cc;
                k_last = k;
            }
            jn = j - 1;
            __syncthreads();
        }
        t_search += clock64() - t_mark;
        if (found || k == max_k) break;
        if (k >= 2) { // the new power becomes X_{k-1}
            uint32_t *tmp = Xp;
            Xp = Xc;
            Xc = tmp;
        } else { // k == 1: X_1 sits in Xa, which Xp already points to
            Xc = Xb;
        }
    }
    if (warp == 0 && lane == 0) flags[5] = dense_from; // (kept by warp 0 only)
    csync(); // no CTA leaves while another may still read its shared memory
    if (rk == 0) { // the result, one element per thread (mapped host memory: one burst of writes)
        const int kk = found ? k_last : k;
        for (int t = tid; t <= kk; t += nthreads) {
            if (t == 0) {
                out[0] = found ? 0 : 4;
                out[1] = mu;
                out[2] = lam;
                out[3] = off;
                out[4] = kk;
                out[5] = flags[5];
            } else {
                out[6 + t] = hs[t].dmin;
                out[6 + (max_k + 1) + t] = (long long)hs[t].fp;
            }
        }
    }
    if (rk == 0 && tid == 0) {
        long long *prof = out + 6 + 2 * (max_k + 1);
        prof[0] = t_setup;
        prof[1] = t_prod;
        prof[2] = t_red;
        prof[3] = t_search;
    }
}

// C column blocks of 64 columns; R row parts (about 56 rows each) as far as a cluster of 16 allows.
static void small_run_shape(int64_t N, int *C, int *R)
{
    *C = (int)((N + 63) / 64);
    *R = (int)std::max<int64_t>(1, std::min<int64_t>(16 / *C, (N + 55) / 56));
}

int small_run_ctas(int64_t N)
{
    int C, R;
    small_run_shape(N, &C, &R);
    return C; // the history pitch is 64 C columns
}

size_t small_run_smem(int64_t N, int R, int max_k, int max_nnz)
{
    const int64_t rows_per = (N + R - 1) / R;
    return (size_t)N * 32 * 4 * 2 + (size_t)rows_per * 8 + (size_t)((rows_per + 4) & ~3) * 4 +
           (size_t)((max_nnz + 1) & ~1) * 8 + (size_t)(max_k + 1 + kSmWarps + 2) * sizeof(Stats) + 2 * 8 + 8 * 4;
}

cudaError_t launch_small_run(const uint16_t *A, int64_t lda, int64_t N, int max_k, int max_nnz, const int32_t *sigma,
                             uint16_t *hist, uint64_t S, long long *out, cudaStream_t s)
{
    if (N < 1 || N > kSmallMaxN) return cudaErrorInvalidValue;
    int C, R;
    small_run_shape(N, &C, &R);
    const size_t smem = small_run_smem(N, R, max_k, max_nnz);
    // per-device kernel attributes: the shared-memory limit (raised to the largest size used)
    // and clusters of up to 16 CTAs (non-portable size)
    static size_t limit[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (limit[dev] < smem) {
        cudaError_t e = cudaFuncSetAttribute(k_small_run, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess) e = cudaFuncSetAttribute(k_small_run, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        limit[dev] = smem;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(C * R));
    // 4 to 16 warps: one row per warp where the rows allow
    const int64_t rows_per = (N + R - 1) / R;
    int warps = (int)std::max<int64_t>(4, std::min<int64_t>(kSmWarps, rows_per)); // a row per warp if possible
    if (const char *e = getenv("MP_SMALL_WARPS")) // experiments: a fixed warp count (1 .. 16)
        warps = std::max(1, std::min(kSmWarps, atoi(e)));
    cfg.blockDim = dim3((unsigned)(32 * warps));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)(C * R);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = C * R > 1 ? 1 : 0; // one CTA: a plain launch (its implicit cluster of one)
    return cudaLaunchKernelEx(&cfg, k_small_run, A, lda, (int)N, C, max_k, max_nnz, sigma, hist,
                              (unsigned long long)S, out);
}

} // namespace mp
