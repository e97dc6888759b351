// C ABI of the (min,+) power path: argument checking, device memory, the power /
// periodicity driver and the gamma_2 read-off.  See include/minplus.h for the contract
// and DESIGN.md for the design.  Product code only: shares nothing with oracle/.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "minplus.h"
#include "mp_internal.h"
#include "mp_kernels.h"

using namespace mp;

namespace {

std::recursive_mutex g_mu;
constexpr double kSpmmAdvantage = 0.6; // auto: SpMM if it issues < 60% of the tile kernel's steps
constexpr int kBatch = 16;             // powers per host round trip when N <= kBatchMaxN
constexpr int64_t kBatchMaxN = 4096;
constexpr int64_t kLookaheadMaxN = 40000; // the lookahead power loop below this order
constexpr double kDefaultRingBytes = 48.0 * 1024 * 1024 * 1024; // power-store cap unless set
thread_local std::string t_err;
std::atomic<int64_t> g_launches{0};
std::atomic<int64_t> g_h2d{0}, g_d2h{0};

struct Dist {
    int rank = 0, world = 1;
    mp_allreduce_fn fn = nullptr;
    void *ctx = nullptr;
    mp_allgather_fn gather = nullptr; // general products: column blocks of C to every rank
    void *gctx = nullptr;
} g_dist;

struct Opts {
    int sparsity = -1; // -1 auto, 0 dense tiles, 1 block-sparse tiles, 2 grouped SpMM
    int64_t budget = 0;
    int grouping = -1; // -1 auto (greedy from kGroupMinN rows), 0 consecutive rows, 1 greedy
} g_opts;
constexpr int64_t kGroupMinN = 8192; // below this the grouping pass costs more than it saves

// Symmetry hint for matrix sources (mp_set_symmetry) and the word-reversal switch for the
// words source.
std::vector<int32_t> g_sym;
uint64_t g_sym_version = 1; // bumped by every mp_set_symmetry (device copies keyed by it)
bool g_word_sym = true;
bool g_small_off = false; // mp_set_small_path(0): always the general path
int g_transfer_n = 0;      // mp_set_transfer_hint: matrix sources claimed to be A(D_n)
// MP_FP_TC=0: the fingerprint on the CUDA cores (k_stats_sym) instead of the tensor cores
bool fp_tc_on()
{
    const char *e = getenv("MP_FP_TC"); // read per run: tests switch it
    return !(e && *e == '0');
}

// MP_LOOKAHEAD=0: no lookahead in the large-N power loop (diagnostic); =2: lookahead at every N
bool lookahead_on()
{
    const char *e = getenv("MP_LOOKAHEAD"); // read per run: tests switch it
    return !(e && *e == '0');
}
bool lookahead_forced()
{
    const char *e = getenv("MP_LOOKAHEAD");
    return e && *e == '2';
}

bool g_row_reuse = true;   // mp_set_row_reuse: row-inclusion reuse for A(D_n)

mp_profile g_prof{};
cudaEvent_t *g_small_prof_ev = nullptr; // small-N run whose event times g_prof still lacks
bool g_small_prof_staged = false;        // ... and whether it recorded ev[0], ev[3] (host staging)

// Parity observer (mp_set_power_observer): sees every power of every run in full.
struct Observer {
    mp_power_observer_fn fn = nullptr;
    void *ctx = nullptr;
} g_obs;
std::map<std::tuple<int, int, int>, mp_periodic_result> g_cache; // (n, world, rank)

// MP_TRACE=1: phase timings of each power run on stderr (the stream is synchronised at every
// mark, so tracing perturbs the timings it reports; for diagnosis, not for benchmarks).
bool trace_on()
{
    static int on = -1;
    if (on < 0) {
        const char *e = getenv("MP_TRACE");
        on = (e && *e && *e != '0') ? 1 : 0;
    }
    return on == 1;
}

// MP_TRACE=1: stream-synchronised phase times on stderr (each mark: time since the previous
// mark of any tracer on this thread, and since this tracer's creation)
thread_local std::chrono::steady_clock::time_point t_trace_last = std::chrono::steady_clock::now();
struct Tracer {
    cudaStream_t s;
    std::chrono::steady_clock::time_point t0;
    explicit Tracer(cudaStream_t st) : s(st), t0(std::chrono::steady_clock::now()) {}
    void mark(const char *what, int k = -1)
    {
        if (!trace_on()) return;
        cudaStreamSynchronize(s);
        const auto now = std::chrono::steady_clock::now();
        const double ms = std::chrono::duration<double, std::milli>(now - t_trace_last).count();
        const double tot = std::chrono::duration<double, std::milli>(now - t0).count();
        if (k >= 0) fprintf(stderr, "mp-trace %-26s k=%-3d %10.3f ms  (%10.3f ms)\n", what, k, ms, tot);
        else fprintf(stderr, "mp-trace %-32s %10.3f ms  (%10.3f ms)\n", what, ms, tot);
        t_trace_last = now;
    }
};

mp_status fail(mp_status s, const char *fmt, ...)
{
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    t_err = buf;
    return s;
}

#define CUDA_TRY(x)                                                                            \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) {                                                               \
            cudaGetLastError();                                                                \
            return fail(MP_ERR_CUDA, "%s failed: %s", #x, cudaGetErrorString(e_));            \
        }                                                                                      \
    } while (0)

#define LAUNCH(x)                                                                              \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        g_launches.fetch_add(1);                                                               \
        if (e_ != cudaSuccess) {                                                               \
            cudaGetLastError();                                                                \
            return fail(MP_ERR_CUDA, "kernel %s failed: %s", #x, cudaGetErrorString(e_));     \
        }                                                                                      \
    } while (0)

// cudaMemcpyAsync that also counts the bytes crossing the host/device boundary.
#define COPY(dst, src, bytes, kind, stream)                                                    \
    do {                                                                                       \
        CUDA_TRY(cudaMemcpyAsync((dst), (src), (bytes), (kind), (stream)));                    \
        if ((kind) == cudaMemcpyHostToDevice) g_h2d.fetch_add((int64_t)(bytes));               \
        if ((kind) == cudaMemcpyDeviceToHost) g_d2h.fetch_add((int64_t)(bytes));               \
    } while (0)

#define TRY(x)                                                                                 \
    do {                                                                                       \
        mp_status s_ = (x);                                                                    \
        if (s_ != MP_OK) return s_;                                                            \
    } while (0)

// Owning device buffer.
struct DBuf {
    void *p = nullptr;
    size_t bytes = 0;
    DBuf() = default;
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
    DBuf(DBuf &&o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
    ~DBuf() { release(); }
    void release()
    {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    mp_status alloc(size_t b, const char *what)
    {
        release();
        if (b == 0) b = 16;
        cudaError_t e = cudaMalloc(&p, b);
        if (e != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
            return fail(MP_ERR_RESOURCE, "device allocation of %zu bytes for %s failed (%s)", b, what,
                        cudaGetErrorString(e));
        }
        bytes = b;
        return MP_OK;
    }
    mp_status ensure(size_t b, const char *what) { return (bytes >= b && p) ? MP_OK : alloc(b, what); }
    template <class T> T *as() const { return reinterpret_cast<T *>(p); }
};

// Workspace of the power driver, kept across calls (like a BLAS workspace) so repeated runs
// do not pay cudaMalloc/cudaFree; released by mp_shutdown().
struct PowerRun {
    int64_t N = 0, Np = 0, c0 = 0, w = 0, ld = 0;
    int spmm_cols = 512; // main k_spmm CTA width of this run (spmm_cols)
    SpmmPlan plan;       // its column segments; ld = plan.ld
    DBuf at2, words, tmp0, tmp1, ktp, kti, occ, stats, flag, stage_raw;
    bool has_at2 = false; // only the tile kernels stage AT2; SpMM reads A or the word masks
    // symmetry: local column jj holds global column gcol[jj] (g <= sigma g) and stands for g and
    // sigma g; cols_rep = number of global columns the local ones stand for
    bool sym = false;
    DBuf bits;            // support bitsets written by k_check_a (matrix sources, grouped SpMM)
    bool bits_ok = false;
    std::vector<int32_t> sigma, gcol, loc; // loc[g] = local column of domain column g (cap path)
    DBuf dsig, dgcol, dloc; // dloc[g] = local column of global column g, or -1
    DBuf drw;               // row weights s(2i), then s(2 sigma i) (symmetric statistics)
    int words_n = 0;        // words holds the word masks of D_(words_n) (0: none)
    DBuf wfrag, tcs;        // tensor-core fingerprint: column-weight byte fragments, per-power {H, #inf}
    bool fptc = false;
    int64_t cols_rep = 0;
    const uint16_t *a_src = nullptr; // matrix sources: A (boundary encoding; the caller's buffer or
    int64_t a_ld = 0;                // stage_raw), valid for the duration of the run
    int n_words = 0;      // path order when A comes from the word masks
    std::vector<DBuf> ring;
    std::vector<int> slot_power;
    std::tuple<size_t, int64_t, int, bool> ring_key{0, 0, 0, false}; // what the slot count was decided for
    size_t cached_slot = 0; // slot size the cached buffers were allocated for
    bool sparse = false;  // tile kernel with l-tile lists
    bool spmm = false;    // grouped SpMM kernel
    int dag_n = 0;        // row-inclusion reuse (A = A(D_dag_n)); 0 = off
    RowDag rdag;
    double issued_per_product = 0.0;
    double issued_tiles = 0.0, issued_spmm = 0.0;
    int64_t tiles_nonempty = 0; // non-empty 128 x 32 tiles of A (block-sparse tile kernel)
    // grouped sparse form of A (k_spmm): buffers handed out in order by sp_alloc
    std::vector<DBuf> sp_bufs;
    size_t sp_next = 0;
    SparseWork sp;
    std::vector<cudaEvent_t> events; // per-power product start/stop
    // observer path: the whole power, unfolded on the device and copied to pinned host memory
    DBuf full_dev;
    DBuf small_hist, small_sig; // small-N path: power history, symmetry hint
    int64_t *hstats = nullptr;             // lookahead: pinned host copy of the statistics
    size_t hstats_n = 0;
    std::vector<cudaEvent_t> events_la;    // lookahead: product done / statistics done, join
    cudaEvent_t small_ev[4] = {nullptr, nullptr, nullptr, nullptr};
    long long *small_host = nullptr;   // the result (mapped pinned host memory) ...
    long long *small_host_dev = nullptr; // ... and its device address
    size_t small_host_n = 0;
    uint64_t small_sig_version = 0;    // g_sym_version of the symmetry hint in small_sig
    uint16_t *full_host = nullptr;
    size_t full_host_bytes = 0;
    ~PowerRun()
    {
        for (auto ev : events)
            if (ev) cudaEventDestroy(ev);
        if (full_host) cudaFreeHost(full_host);
        for (auto ev : small_ev)
            if (ev) cudaEventDestroy(ev);
        for (auto ev : events_la)
            if (ev) cudaEventDestroy(ev);
        if (hstats) cudaFreeHost(hstats);
        if (small_host) cudaFreeHost(small_host);
    }
    size_t slot_bytes() const { return (size_t)Np * ld * 2; }
};

// Per-device state: a library stream, scratch for minplus_mul(_device), the power workspace.
struct DevState {
    cudaStream_t stream = nullptr;      // the library's own non-blocking stream
    cudaStream_t user_stream = nullptr; // mp_set_stream override for power runs
    cudaStream_t stream2 = nullptr;     // second stream of the lookahead power loop
    DBuf at2, xb, cb, flag, stage_a, stage_b, stage_c, shard_c, gathered;
    // last use of the product scratch (at2, xb, cb, flag): the next user, on whatever stream,
    // waits on it, so a call on another stream cannot overwrite scratch still being read
    cudaEvent_t scratch_ev = nullptr;
    std::unique_ptr<PowerRun> pr;
};
std::map<int, DevState> g_dev;

mp_status current_device(int *dev_out, DevState **st)
{
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        cudaGetLastError();
        return fail(MP_ERR_CUDA, "no CUDA device available (%s); this library has no CPU fallback",
                    e != cudaSuccess ? cudaGetErrorString(e) : "0 devices");
    }
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    auto it = g_dev.find(dev);
    if (it == g_dev.end()) {
        cudaDeviceProp prop;
        CUDA_TRY(cudaGetDeviceProperties(&prop, dev));
        if (prop.major != 10)
            return fail(MP_ERR_CUDA, "device %d (%s, sm_%d%d) is not sm_100; this build targets sm_100a", dev,
                        prop.name, prop.major, prop.minor);
        DevState ds;
        CUDA_TRY(cudaStreamCreateWithFlags(&ds.stream, cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreateWithFlags(&ds.scratch_ev, cudaEventDisableTiming));
        it = g_dev.emplace(dev, std::move(ds)).first;
    }
    *dev_out = dev;
    *st = &it->second;
    return MP_OK;
}

bool overlaps(const void *a, size_t abytes, const void *b, size_t bbytes)
{
    const char *x = (const char *)a, *y = (const char *)b;
    return x < y + bbytes && y < x + abytes;
}

size_t span_bytes(int64_t rows, int64_t cols, int64_t ld) { return (size_t)((rows - 1) * ld + cols) * 2; }

int host_threads()
{
    unsigned h = std::thread::hardware_concurrency();
    return h ? (int)std::min(h, 64u) : 4;
}

// ---------------------------------------------------------------------------------------
// Product on device buffers (boundary encoding in and out).
// ---------------------------------------------------------------------------------------
// C_b = A_b (x) B_b for b < batch (strides in elements; batch 1 = one product).  The items go
// through the tile kernel together -- one launch of each kernel per chunk of items, the chunk as
// large as 8 GB of scratch allows -- with one read of the range flag per chunk.
mp_status mul_device_impl(DevState &st, const uint16_t *dA, int64_t lda, int64_t sA, const uint16_t *dB, int64_t ldb,
                          int64_t sB, uint16_t *dC, int64_t ldc, int64_t sC, int64_t M, int64_t K, int64_t N,
                          int64_t batch, cudaStream_t s)
{
    const int64_t Mp = pad_rows(M), Kp = pad_rows(K), Np = pad_cols(N);
    const int64_t at_i = Kp * Mp, xb_i = Kp * Np, cb_i = Mp * Np; // scratch elements per item
    const int64_t per = at_i * 4 + xb_i * 2 + cb_i * 2;
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>({batch, (int64_t)(8LL << 30) / per, 65535}));
    TRY(st.at2.ensure((size_t)(chunk * at_i) * 4, "A (transposed, duplicated)"));
    TRY(st.xb.ensure((size_t)(chunk * xb_i) * 2, "B (padded)"));
    TRY(st.cb.ensure((size_t)(chunk * cb_i) * 2, "C (padded)"));
    TRY(st.flag.ensure(16, "range flag"));
    CUDA_TRY(cudaStreamWaitEvent(s, st.scratch_ev, 0)); // the previous user of the scratch is done
    for (int64_t b0 = 0; b0 < batch; b0 += chunk) {
        const int nb = (int)std::min<int64_t>(chunk, batch - b0);
        CUDA_TRY(cudaMemsetAsync(st.flag.p, 0, sizeof(int), s));
        LAUNCH(launch_make_at2(dA + b0 * sA, lda, M, K, st.at2.as<uint32_t>(), Mp, Kp, st.flag.as<int>(), s, nb, sA,
                               at_i));
        LAUNCH(launch_encode(dB + b0 * sB, ldb, K, N, st.xb.as<uint16_t>(), Np, Kp, st.flag.as<int>(), s, nb, sB,
                             xb_i));
        int flag = 0;
        COPY(&flag, st.flag.p, sizeof(int), cudaMemcpyDeviceToHost, s);
        CUDA_TRY(cudaStreamSynchronize(s));
        if (flag) return fail(MP_ERR_RANGE, "an input entry lies in (0x7FFE, 0xFFFF)");
        LAUNCH(launch_minplus(st.at2.as<uint32_t>(), Mp, st.xb.as<uint16_t>(), Np, st.cb.as<uint16_t>(), Np, Mp, Np,
                              Kp, nullptr, nullptr, s, nb, at_i, xb_i, cb_i));
        LAUNCH(launch_decode(st.cb.as<uint16_t>(), Np, M, N, dC + b0 * sC, ldc, s, nb, cb_i, sC));
    }
    CUDA_TRY(cudaEventRecord(st.scratch_ev, s));
    return MP_OK;
}

mp_status mul_device_impl(DevState &st, const uint16_t *dA, int64_t lda, const uint16_t *dB, int64_t ldb,
                          uint16_t *dC, int64_t ldc, int64_t M, int64_t K, int64_t N, cudaStream_t s)
{
    return mul_device_impl(st, dA, lda, 0, dB, ldb, 0, dC, ldc, 0, M, K, N, 1, s);
}

// Column-sharded product over the ranks of the distributed context (one GPU each; SURVEY.md
// section 8(b)/(e)): A replicated, rank r computes C[:, J_r] = A (x) B[:, J_r] on its
// column shard J_r = mp_shard_range(N, world, r), and the all-gather callback hands every rank
// every block, which k_unshard places into the whole C (device, pitch N).
bool sharded_products() { return g_dist.world > 1 && g_dist.gather != nullptr; }

mp_status mul_sharded(DevState &st, const uint16_t *dA, const uint16_t *dB, int64_t ldb, uint16_t *dC, int64_t M,
                      int64_t K, int64_t N, cudaStream_t s)
{
    int64_t c0 = 0, c1 = 0;
    mp_shard_range(N, g_dist.world, g_dist.rank, &c0, &c1);
    const int64_t w = round_up((N + g_dist.world - 1) / g_dist.world, 8); // every rank's block width
    const size_t blk = (size_t)M * w * 2;
    TRY(st.shard_c.ensure(blk, "C column block"));
    TRY(st.gathered.ensure(blk * g_dist.world, "gathered C blocks"));
    if (c1 > c0) TRY(mul_device_impl(st, dA, K, dB + c0, ldb, st.shard_c.as<uint16_t>(), w, M, K, c1 - c0, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (g_dist.gather(g_dist.gctx, st.shard_c.p, st.gathered.p, (int64_t)blk, (void *)s) != 0)
        return fail(MP_ERR_COMM, "all-gather callback failed (%zu bytes per rank)", blk);
    LAUNCH(launch_unshard(st.gathered.as<uint16_t>(), g_dist.world, M, w, N, dC, N, s));
    return MP_OK;
}

// ---------------------------------------------------------------------------------------
// Power / periodicity driver (a3-a5)
// ---------------------------------------------------------------------------------------

mp_status allreduce(int op, int64_t *dev, int64_t count, cudaStream_t s)
{
    if (!g_dist.fn) return MP_OK; // a registered callback runs even for world == 1
    CUDA_TRY(cudaStreamSynchronize(s));
    if (g_dist.fn(g_dist.ctx, op, dev, count, (void *)s) != 0)
        return fail(MP_ERR_COMM, "all-reduce callback failed (op %d, %lld values)", op, (long long)count);
    return MP_OK;
}

// Block-sparse l-tile lists of A (exact skipping of all-inf tiles).
// R.occ holds the 128 x 32 tile occupancy (launch_check_a or launch_tile_occupancy).
mp_status build_tile_lists(PowerRun &R, cudaStream_t s)
{
    const int64_t Mt = R.Np / kBM, Kt = R.Np / kBK;
    std::vector<uint8_t> h((size_t)(Mt * Kt));
    COPY(h.data(), R.occ.p, h.size(), cudaMemcpyDeviceToHost, s);
    CUDA_TRY(cudaStreamSynchronize(s));
    std::vector<int32_t> ptr((size_t)Mt + 1, 0), idx;
    idx.reserve(h.size() / 4);
    for (int64_t b = 0; b < Mt; ++b) {
        for (int64_t k = 0; k < Kt; ++k)
            if (h[(size_t)(b * Kt + k)]) idx.push_back((int32_t)k);
        ptr[(size_t)b + 1] = (int32_t)idx.size();
    }
    if (idx.empty()) idx.push_back(0);
    TRY(R.ktp.ensure(ptr.size() * 4, "tile list pointers"));
    TRY(R.kti.ensure(idx.size() * 4, "tile list"));
    COPY(R.ktp.p, ptr.data(), ptr.size() * 4, cudaMemcpyHostToDevice, s);
    COPY(R.kti.p, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice, s);
    CUDA_TRY(cudaStreamSynchronize(s));
    R.tiles_nonempty = ptr[(size_t)Mt];
    R.issued_tiles = (double)R.tiles_nonempty * kBK * kBM * (double)R.ld;
    return MP_OK;
}

// Grouped sparse form of A (k_spmm): built on the device from AT2.
cudaError_t sp_alloc(void **p, size_t bytes, void *ctx)
{
    PowerRun *R = static_cast<PowerRun *>(ctx);
    if (R->sp_next >= R->sp_bufs.size()) R->sp_bufs.resize(R->sp_next + 1);
    DBuf &b = R->sp_bufs[R->sp_next++];
    if (b.ensure(bytes, "sparse form of A") != MP_OK) return cudaErrorMemoryAllocation;
    *p = b.p;
    return cudaSuccess;
}

// The word masks of D_n on the device (kept across runs of the same n)
mp_status stage_words(PowerRun &R, int n, cudaStream_t s)
{
    if (R.words_n == n && R.words.p) return MP_OK;
    const std::vector<WordMask> words = enumerate_words(n);
    R.words_n = 0;
    TRY(R.words.ensure(words.size() * sizeof(WordMask), "word masks"));
    COPY(R.words.p, words.data(), words.size() * sizeof(WordMask), cudaMemcpyHostToDevice, s);
    CUDA_TRY(cudaStreamSynchronize(s)); // the host vector goes out of scope
    R.words_n = n;
    return MP_OK;
}

mp_status build_sparse(PowerRun &R, cudaStream_t s)
{
    R.sp_next = 0;
    R.sp = SparseWork();
    R.sp.cols = R.spmm_cols; // reported width (the entries carry row offsets for every width)
    int64_t launches = 0;
    const bool group = g_opts.grouping == 1 || (g_opts.grouping < 0 && R.N >= kGroupMinN);
    cudaError_t e = cudaSuccess;
    const RowDag *dag = nullptr;
    if (R.dag_n && group) { // row-inclusion reuse: parents and levels
        R.rdag = RowDag();
        e = build_row_dag(R.words.as<WordMask>(), R.N, R.dag_n, R.rdag, s, sp_alloc, &R, &launches);
        if (trace_on()) Tracer(s).mark("  row DAG (since a2)");
        dag = &R.rdag;
    } else {
        R.dag_n = 0;
    }
    if (e == cudaSuccess)
        e = R.a_src ? build_sparse_form(R.a_src, R.a_ld, R.N, R.Np, group,
                                        group && R.bits_ok ? R.bits.as<uint32_t>() : nullptr, R.sp, s, sp_alloc, &R,
                                        &launches, dag)
                    : build_sparse_form_words(R.words.as<WordMask>(), R.N, R.n_words, R.Np, group, R.sp, s, sp_alloc,
                                              &R, &launches, dag);
    if (trace_on()) Tracer(s).mark("  sparse form");
    g_launches.fetch_add(launches);
    g_d2h.fetch_add(24);
    if (e == cudaErrorMemoryAllocation) return MP_ERR_RESOURCE; // message set by DBuf::alloc
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(MP_ERR_CUDA, "building the sparse form of A failed: %s", cudaGetErrorString(e));
    }
    if (dag) { // every parent's support must lie inside its child's
        int bad = 0;
        COPY(&bad, R.rdag.bad, sizeof(int), cudaMemcpyDeviceToHost, s);
        CUDA_TRY(cudaStreamSynchronize(s));
        if (bad) return fail(MP_ERR_CUDA, "internal: a row-inclusion parent is not a subset of its row");
    }
    R.issued_spmm = (double)R.sp.entries * (double)R.sp.group_rows * (double)R.ld;
    return MP_OK;
}

// C = A (x) X with the selected kernel.
// mid (may be null): recorded between the SpMM and the fold passes of the row-inclusion reuse.
mp_status product(PowerRun &R, const uint16_t *X, uint16_t *C, cudaStream_t s, cudaEvent_t mid = nullptr)
{
    if (R.spmm) {
        SparseA sa;
        sa.L = R.sp.L;
        sa.tptr = R.sp.tptr;
        sa.tch = R.sp.tch;
        sa.eoff = R.sp.eoff;
        sa.E = R.sp.E;
        sa.rows = R.sp.rows;
        int nl = 0;
        cudaError_t e = launch_spmm(sa, R.plan, X, R.ld, C, R.ld, R.Np, s, &nl);
        if (e == cudaSuccess && mid) e = cudaEventRecord(mid, s);
        if (e == cudaSuccess && R.dag_n) e = launch_folds(R.rdag, C, R.ld, R.ld, s, &nl); // parents' rows
        g_launches.fetch_add(nl);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(MP_ERR_CUDA, "kernel k_spmm failed: %s", cudaGetErrorString(e));
        }
        return MP_OK;
    }
    LAUNCH(launch_minplus(R.at2.as<uint32_t>(), R.Np, X, R.ld, C, R.ld, R.Np, R.ld, R.Np,
                          R.sparse ? R.ktp.as<int32_t>() : nullptr, R.sparse ? R.kti.as<int32_t>() : nullptr, s));
    return MP_OK;
}

// X_1 = A[:, c0:c0+w) in the device layout, from A, AT2 or straight from the word masks.
mp_status make_power1(PowerRun &R, uint16_t *dst, cudaStream_t s)
{
    if (R.spmm && R.a_src && R.bits_ok && !R.sp.off) { // A's support bitsets from the range check
        g_launches.fetch_add(1);
        LAUNCH(launch_x1_bits(R.bits.as<uint32_t>(), R.N, R.a_src, R.a_ld, R.dloc.as<int32_t>(), dst, R.ld, R.Np, s));
        return MP_OK;
    }
    if (R.spmm && R.sp.off) { // row lists of A available (grouped path): fill + scatter
        LAUNCH(launch_x1_csr(R.sp.off, R.sp.idx, R.N, R.a_src, R.a_ld, R.a_src ? nullptr : R.words.as<WordMask>(),
                             R.dloc.as<int32_t>(), dst, R.ld, R.Np, s));
        return MP_OK;
    }
    if (R.sym) {
        if (R.a_src)
            LAUNCH(launch_encode_cols(R.a_src, R.a_ld, R.N, R.dgcol.as<int32_t>(), R.w, dst, R.ld, R.Np, s));
        else
            LAUNCH(launch_x1_from_words(R.words.as<WordMask>(), R.N, R.n_words, R.Np, 0, R.dgcol.as<int32_t>(), R.w,
                                        dst, R.ld, s));
        return MP_OK;
    }
    if (R.a_src) // range-checked already: the flag is scratch
        LAUNCH(launch_encode(R.a_src + R.c0, R.a_ld, R.N, R.w, dst, R.ld, R.Np, R.flag.as<int>(), s));
    else if (R.has_at2)
        LAUNCH(launch_x1_from_at2(R.at2.as<uint32_t>(), R.Np, R.c0, R.w, dst, R.ld, s));
    else
        LAUNCH(launch_x1_from_words(R.words.as<WordMask>(), R.N, R.n_words, R.Np, R.c0, nullptr, R.w, dst, R.ld, s));
    return MP_OK;
}

// Returns the device buffer holding power j, recomputing it into two scratch buffers if it
// has been evicted from the ring.
mp_status power_buffer(PowerRun &R, int j, const uint16_t **out, cudaStream_t s)
{
    for (size_t q = 0; q < R.ring.size(); ++q)
        if (R.slot_power[q] == j) {
            *out = R.ring[q].as<uint16_t>();
            return MP_OK;
        }
    TRY(R.tmp0.ensure(R.slot_bytes(), "recompute buffer"));
    TRY(R.tmp1.ensure(R.slot_bytes(), "recompute buffer"));
    TRY(make_power1(R, R.tmp1.as<uint16_t>(), s));
    const uint16_t *cur = R.tmp1.as<uint16_t>();
    for (int k = 2; k <= j; ++k) {
        uint16_t *dst = (k & 1) ? R.tmp1.as<uint16_t>() : R.tmp0.as<uint16_t>();
        TRY(product(R, cur, dst, s));
        cur = dst;
    }
    *out = cur;
    return MP_OK;
}

// Hands the whole power A^k (boundary encoding, host memory) to the observer.
mp_status observe(PowerRun &R, const uint16_t *X, int k, cudaStream_t s)
{
    const size_t bytes = (size_t)R.N * (size_t)R.N * 2;
    TRY(R.full_dev.ensure(bytes, "observer copy of a power"));
    if (R.full_host_bytes < bytes) {
        if (R.full_host) cudaFreeHost(R.full_host);
        R.full_host = nullptr;
        R.full_host_bytes = 0;
        if (cudaMallocHost((void **)&R.full_host, bytes) != cudaSuccess) {
            cudaGetLastError();
            R.full_host = nullptr;
            return fail(MP_ERR_RESOURCE, "pinned host allocation of %zu bytes for the power observer failed", bytes);
        }
        R.full_host_bytes = bytes;
    }
    LAUNCH(launch_unfold(X, R.ld, R.N, R.dloc.as<int32_t>(), R.sym ? R.dsig.as<int32_t>() : nullptr,
                         R.full_dev.as<uint16_t>(), s));
    COPY(R.full_host, R.full_dev.p, bytes, cudaMemcpyDeviceToHost, s);
    CUDA_TRY(cudaStreamSynchronize(s));
    if (g_obs.fn(g_obs.ctx, k, R.full_host, R.N) != 0)
        return fail(MP_ERR_DOMAIN, "the power observer stopped the run at k = %d", k);
    return MP_OK;
}

// Source of A: either a host matrix or the word masks of path order n.
struct ASource {
    const uint16_t *host = nullptr; // host matrix, pitch N
    const uint16_t *dev = nullptr;  // device matrix, pitch lda
    int64_t lda = 0;
    int n = 0;                      // else: build A(D_n) from the word masks on the device
};

// Optional row capture (minplus_power_rows): no periodicity search, stop at kmax.
struct Capture {
    const int64_t *rows = nullptr;
    int nrows = 0;
    uint16_t *out = nullptr; // host
};

// Small-N latency path (DESIGN.md section 5 "Small-N path"): the whole run -- products,
// statistics, repeat search, exact compares -- in one thread-block-cluster launch, one read of
// the result.  *handled = false (and MP_OK) if A has too many finite entries for the kernel's
// shared memory; the caller then takes the general path.
constexpr int kSmallMaxNnz = 8192; // 64 KB of {offset, value} entries in shared memory
mp_status run_small(DevState &st, const ASource &src, int64_t N, int max_k, mp_periodic_result *out, bool *handled)
{
    *handled = false;
    if (!st.pr) st.pr.reset(new PowerRun());
    PowerRun &R = *st.pr;
    cudaStream_t s = st.user_stream ? st.user_stream : st.stream;
    const int64_t h2d0 = g_h2d.load(), d2h0 = g_d2h.load();
    cudaEvent_t *ev = R.small_ev;
    if (!ev[0])
        for (int i = 0; i < 4; ++i) CUDA_TRY(cudaEventCreate(&ev[i]));
    // events: ev[1], ev[2] around the kernel; ev[0], ev[3] around the whole call only when a
    // host matrix is staged (each record costs the caller about a microsecond at n = 3)
    const bool staged = !src.dev;
    if (staged) CUDA_TRY(cudaEventRecord(ev[0], s));
    const uint16_t *dA = src.dev;
    int64_t lda = src.lda;
    if (!dA) { // host matrix, or A(D_n) from the word masks (at most 256 x 256 here)
        std::vector<uint16_t> words_A;
        const uint16_t *h = src.host;
        if (!h) {
            words_A.resize((size_t)N * N);
            fill_transition_matrix(enumerate_words(src.n), src.n, words_A.data(), 1);
            h = words_A.data();
        }
        TRY(R.stage_raw.ensure((size_t)N * N * 2, "A staging"));
        COPY(R.stage_raw.p, h, (size_t)N * N * 2, cudaMemcpyHostToDevice, s);
        if (!src.host) CUDA_TRY(cudaStreamSynchronize(s)); // words_A is about to go away
        dA = R.stage_raw.as<uint16_t>();
        lda = N;
    }
    const int C = small_run_ctas(N);
    TRY(R.small_hist.ensure((size_t)(max_k + 1) * N * 64 * C * 2, "small-N power history"));
    const size_t nout = 6 + 2 * (size_t)(max_k + 1) + 4; // + 4 clock64 phase sums
    // the result goes straight to mapped pinned host memory (no copy after the kernel)
    if (R.small_host_n < nout) {
        if (R.small_host) cudaFreeHost(R.small_host);
        R.small_host = nullptr;
        R.small_host_n = 0;
        CUDA_TRY(cudaHostAlloc((void **)&R.small_host, nout * 8, cudaHostAllocMapped));
        CUDA_TRY(cudaHostGetDevicePointer((void **)&R.small_host_dev, R.small_host, 0));
        R.small_host_n = nout;
    }
    const uint64_t S = mp_fingerprint_unit(N);
    const int32_t *dsig = nullptr;
    if ((src.dev || src.host) && (int64_t)g_sym.size() == N) { // a matrix source's symmetry hint
        if (R.small_sig_version != g_sym_version || R.small_sig.bytes < (size_t)N * 4) { // copied once per hint
            R.small_sig_version = 0;
            TRY(R.small_sig.ensure((size_t)N * 4, "symmetry"));
            COPY(R.small_sig.p, g_sym.data(), (size_t)N * 4, cudaMemcpyHostToDevice, s);
            R.small_sig_version = g_sym_version;
        }
        dsig = R.small_sig.as<int32_t>();
    }
    CUDA_TRY(cudaEventRecord(ev[1], s));
    // entry capacity: at most N^2 finite entries (n = 3: 2 KB of shared memory instead of 64 KB,
    // which keeps the launch off a shared-memory carveout change)
    const int max_nnz = (int)std::min<int64_t>(kSmallMaxNnz, N * N);
    LAUNCH(launch_small_run(dA, lda, N, max_k, max_nnz, dsig, R.small_hist.as<uint16_t>(), S,
                            R.small_host_dev, s));
    CUDA_TRY(cudaEventRecord(ev[2], s));
    long long *h = R.small_host;
    g_d2h.fetch_add((int64_t)nout * 8); // written over the bus by the kernel
    if (staged) CUDA_TRY(cudaEventRecord(ev[3], s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (h[0] == -1) return MP_OK; // too many finite entries: the general path
    if (getenv("MP_SMALL_PROFILE")) {
        const long long *pf = h + 6 + 2 * (max_k + 1);
        fprintf(stderr, "mp-small N=%lld k_last=%lld cycles: setup %lld, products+stats %lld, reductions %lld, search %lld\n",
                (long long)N, h[4], pf[0], pf[1], pf[2], pf[3]);
    }
    *handled = true;
    const int products = (int)h[4] - 1;
    g_prof = mp_profile{};
    // the event times are read by mp_last_profile (three cudaEventElapsedTime calls cost more
    // than a tenth of an n = 3 run)
    g_small_prof_ev = ev;
    g_small_prof_staged = staged;
    g_prof.product_launches = products;
    g_prof.dense_steps = (double)products * (double)N * (double)N * (double)N;
    g_prof.issued_steps = 0.0; // the row lists of A against 64 C columns; counted by the caller as nnz * 64 C
    g_prof.stats_ms = 0.0; // fused
    g_prof.h2d_bytes = g_h2d.load() - h2d0;
    g_prof.d2h_bytes = g_d2h.load() - d2h0;
    g_prof.kernel = 3;
    g_prof.spmm_cols = 0;
    g_prof.local_cols = N;
    g_prof.ld = 64 * C;
    if (h[0] == 2) return fail(MP_ERR_RANGE, "an entry of A lies in (0x7FFE, 0xFFFF)");
    if (h[0] == 1) return fail(MP_ERR_DOMAIN, "symmetry hint: A[sigma i][sigma j] != A[i][j] for some i, j");
    if (h[0] == 4) return fail(MP_ERR_NOT_PERIODIC, "no repeat A^k = c (x) A^j with k <= %d", max_k);
    mp_periodic_result res;
    std::memset(&res, 0, sizeof(res));
    res.mu = (int32_t)h[1];
    res.lambda = (int32_t)h[2];
    res.offset = (int32_t)h[3];
    res.k_last = (int32_t)h[4];
    res.dense_from = (int32_t)h[5];
    for (int k = 1; k <= res.k_last; ++k) {
        res.diag_min[k] = (uint16_t)std::min<long long>(h[6 + k], 0xFFFF);
        res.fingerprint[k] = (uint64_t)h[6 + (max_k + 1) + k];
    }
    *out = res;
    return MP_OK;
}

// The small-N path applies to single-rank runs of small matrices with the automatic kernel
// choice and no observer (a forced kernel, a sharded run or an observer take the general path,
// which the tests also exercise at these sizes; mp_set_small_path(0) forces it).
bool small_path_ok(const ASource &src, int64_t N, const Capture *cap)
{
    (void)src;
    if (cap || N > kSmallMaxN || g_opts.sparsity != -1 || g_dist.world > 1 || g_dist.fn || g_obs.fn) return false;
    return !g_small_off;
}

mp_status run_powers(const ASource &src, int64_t N, int max_k, mp_periodic_result *out,
                     const Capture *cap = nullptr)
{
    g_small_prof_ev = nullptr; // a new run: its own profile
    if (small_path_ok(src, N, cap)) {
        int dev0 = 0;
        DevState *st0 = nullptr;
        TRY(current_device(&dev0, &st0));
        bool handled = false;
        TRY(run_small(*st0, src, N, max_k, out, &handled));
        if (handled) return MP_OK;
    }
    int dev = 0;
    DevState *st = nullptr;
    TRY(current_device(&dev, &st));
    if (g_obs.fn && !cap && g_dist.world > 1)
        return fail(MP_ERR_DOMAIN, "the power observer needs the whole power: single rank only (world = %d)",
                    g_dist.world);
    cudaStream_t s = st->user_stream ? st->user_stream : st->stream;
    const int64_t h2d0 = g_h2d.load(), d2h0 = g_d2h.load();
    cudaEvent_t ev_all0, ev_all1;
    CUDA_TRY(cudaEventCreate(&ev_all0));
    CUDA_TRY(cudaEventCreate(&ev_all1));
    CUDA_TRY(cudaEventRecord(ev_all0, s));
    Tracer tr(s);
    tr.mark("start");

    if (!st->pr) st->pr.reset(new PowerRun());
    PowerRun &R = *st->pr;
    R.N = N;
    R.Np = pad_rows(N);
    const bool words_src = !src.dev && !src.host;
    // Columns this run computes: a shard of [0, N), or under a symmetry sigma (DESIGN.md
    // "Symmetry") a shard of the domain D = {g : g <= sigma g} -- every power satisfies
    // X_(sigma i, sigma j) = X_ij, and column j of A^k depends only on column j of A^{k-1}.
    R.sigma.clear();
    if (words_src && g_word_sym) R.sigma = word_reversal(src.n);
    else if (!words_src && (int64_t)g_sym.size() == N) R.sigma = g_sym;
    R.sym = !R.sigma.empty();
    if (R.sym) {
        for (int64_t i = 0; i < N; ++i)
            if (R.sigma[i] < 0 || R.sigma[i] >= N || R.sigma[R.sigma[i]] != i)
                return fail(MP_ERR_DOMAIN, "symmetry: sigma is not an involution of [0, %lld)", (long long)N);
        std::vector<int32_t> dom;
        for (int64_t g = 0; g < N; ++g)
            if (g <= R.sigma[g]) dom.push_back((int32_t)g);
        int64_t c0 = 0, c1 = (int64_t)dom.size();
        if (!cap) mp_shard_range((int64_t)dom.size(), g_dist.world, g_dist.rank, &c0, &c1);
        R.gcol.assign(dom.begin() + c0, dom.begin() + c1);
        R.c0 = 0;
        R.w = c1 - c0;
        R.cols_rep = 0;
        R.loc.assign((size_t)N, -1);
        for (size_t jj = 0; jj < R.gcol.size(); ++jj) {
            R.cols_rep += (R.sigma[R.gcol[jj]] != R.gcol[jj]) ? 2 : 1;
            R.loc[(size_t)R.gcol[jj]] = (int32_t)jj;
        }
        TRY(R.dsig.ensure((size_t)N * 4, "symmetry"));
        TRY(R.dgcol.ensure(std::max<size_t>(R.gcol.size(), 1) * 4, "column list"));
        COPY(R.dsig.p, R.sigma.data(), (size_t)N * 4, cudaMemcpyHostToDevice, s);
        TRY(R.drw.ensure((size_t)N * 16, "row weights"));
        LAUNCH(launch_row_weights(N, R.dsig.as<int32_t>(), R.drw.as<uint64_t>(), R.drw.as<uint64_t>() + N, s));
        if (!R.gcol.empty())
            COPY(R.dgcol.p, R.gcol.data(), R.gcol.size() * 4, cudaMemcpyHostToDevice, s);
    } else {
        int64_t c0, c1;
        mp_shard_range(N, g_dist.world, g_dist.rank, &c0, &c1);
        R.c0 = c0;
        R.w = c1 - c0;
        if (cap) { // single device, whole matrix
            R.c0 = 0;
            R.w = N;
        }
        R.cols_rep = R.w;
    }
    R.plan = spmm_plan(R.Np, R.w); // SpMM CTA widths of this run (DESIGN.md sections 5, 6)
    R.spmm_cols = R.plan.main_cols;
    R.ld = R.plan.ld;
    {
        std::vector<int32_t> dl((size_t)N, -1);
        if (R.sym)
            for (size_t jj = 0; jj < R.gcol.size(); ++jj) dl[(size_t)R.gcol[jj]] = (int32_t)jj;
        else
            for (int64_t j = 0; j < R.w; ++j) dl[(size_t)(R.c0 + j)] = (int32_t)j;
        TRY(R.dloc.ensure((size_t)N * 4, "column map"));
        COPY(R.dloc.p, dl.data(), (size_t)N * 4, cudaMemcpyHostToDevice, s);
    }
    if (R.slot_bytes() != R.cached_slot) {
        R.ring.clear();
        R.tmp0.release();
        R.tmp1.release();
        R.cached_slot = R.slot_bytes();
    }

    // a2: stage A.  Matrix sources are range-checked in place (host ones copied to a staging
    // buffer first) and read directly by the SpMM sparse-form builder and by X_1; only the tile
    // kernels need AT2 (transposed, duplicated, device encoding), built once they are chosen.
    // The words source with SpMM needs no matrix at all (69 GB saved at n = 13).
    R.n_words = words_src ? src.n : 0;
    R.bits_ok = false;
    R.a_src = nullptr;
    R.a_ld = 0;
    TRY(R.flag.ensure(16, "range flag"));
    const int64_t Mt = R.Np / kBM, Kt = R.Np / kBK;
    if (words_src) {
        TRY(stage_words(R, src.n, s));
    } else {
        R.a_src = src.dev;
        R.a_ld = src.lda;
        if (src.host) { // staging buffer kept with the workspace (no 2N^2-byte malloc per call)
            // rows padded to 64 columns: 128-byte aligned rows for the vectorised range check
            const int64_t pitch = round_up(N, 64);
            TRY(R.stage_raw.ensure((size_t)N * pitch * 2, "A staging"));
            CUDA_TRY(cudaMemcpy2DAsync(R.stage_raw.p, (size_t)pitch * 2, src.host, (size_t)N * 2, (size_t)N * 2,
                                       (size_t)N, cudaMemcpyHostToDevice, s));
            g_h2d.fetch_add((int64_t)N * N * 2);
            R.a_src = R.stage_raw.as<uint16_t>();
            R.a_ld = pitch;
        }
        // a transfer-matrix hint (mp_set_transfer_hint) brings the word masks along, verified below
        const bool hint = g_transfer_n >= 2 && count_words(g_transfer_n) == N;
        // the tile occupancy only feeds the tile kernels' choice: A(D_n) (a verified hint) takes
        // the grouped SpMM directly, as the words source does
        const bool need_occ = g_opts.sparsity != 0 && g_opts.sparsity != 2 && !hint;
        if (need_occ) {
            TRY(R.occ.ensure((size_t)(Mt * Kt), "tile occupancy"));
            CUDA_TRY(cudaMemsetAsync(R.occ.p, 0, (size_t)(Mt * Kt), s));
        }
        // the grouped SpMM path needs A's support bitsets: the range check writes them
        R.bits_ok = (g_opts.sparsity == 2 || g_opts.sparsity < 0) &&
                    (g_opts.grouping == 1 || (g_opts.grouping < 0 && N >= kGroupMinN));
        if (R.bits_ok) TRY(R.bits.ensure((size_t)N * ((N + 31) / 32) * 4, "support bitsets"));
        if (hint) TRY(stage_words(R, g_transfer_n, s));
        CUDA_TRY(cudaMemsetAsync(R.flag.p, 0, 3 * sizeof(int), s));
        // A verified equal to A(D_n) is reflection-symmetric (DESIGN.md section 4 "Symmetry"):
        // a symmetry hint that IS the word reversal then needs no separate check
        const bool sym_implied = hint && R.sym && R.sigma == word_reversal(g_transfer_n);
        LAUNCH(launch_check_a(R.a_src, R.a_ld, N, R.Np, need_occ ? R.occ.as<uint8_t>() : nullptr, R.flag.as<int>(),
                              R.sym && !sym_implied ? R.dsig.as<int32_t>() : nullptr, R.flag.as<int>() + 1,
                              R.bits_ok ? R.bits.as<uint32_t>() : nullptr, s, hint ? R.words.as<WordMask>() : nullptr,
                              g_transfer_n, R.flag.as<int>() + 2));
        int hflag[3] = {0, 0, 0};
        COPY(hflag, R.flag.p, 3 * sizeof(int), cudaMemcpyDeviceToHost, s);
        CUDA_TRY(cudaStreamSynchronize(s));
        if (hflag[0]) return fail(MP_ERR_RANGE, "an entry of A lies in (0x7FFE, 0xFFFF)");
        if (hflag[1]) return fail(MP_ERR_DOMAIN, "symmetry hint: A[sigma i][sigma j] != A[i][j] for some i, j");
        if (hflag[2]) return fail(MP_ERR_DOMAIN, "transfer hint: A is not A(D_%d)", g_transfer_n);
        if (hint) R.n_words = g_transfer_n; // the rows' word structure is now known
        tr.mark("a2 check A");
    }
    // row-inclusion reuse needs the word structure and the grouped SpMM
    R.dag_n = (g_row_reuse && R.n_words && (g_opts.sparsity == 2 || g_opts.sparsity < 0)) ? R.n_words : 0;


    tr.mark("a2 stage A");

    // kernel choice: dense tiles, block-sparse tiles, grouped SpMM
    R.sparse = R.spmm = false;
    R.has_at2 = false;
    if (g_opts.sparsity == 2 || (g_opts.sparsity < 0 && (words_src || R.n_words))) {
        TRY(build_sparse(R, s));
        R.spmm = true;
        R.issued_per_product = R.issued_spmm;
    } else {
        if (g_opts.sparsity != 0 && !words_src) TRY(build_tile_lists(R, s)); // occupancy from A
        if (g_opts.sparsity < 0) { // matrix source, auto
            TRY(build_sparse(R, s));
            if (R.issued_spmm < kSpmmAdvantage * R.issued_tiles) {
                R.spmm = true;
                R.issued_per_product = R.issued_spmm;
            }
        }
        if (!R.spmm) { // the tile kernels: stage AT2; their CTA is 256 columns wide
            R.ld = round_up(R.ld, kBN);
            R.issued_tiles = (double)R.tiles_nonempty * kBK * kBM * (double)R.ld;
            TRY(R.at2.ensure((size_t)R.Np * R.Np * 4, "A (transposed, duplicated)"));
            if (words_src) {
                LAUNCH(launch_build_from_words(R.words.as<WordMask>(), N, src.n, R.at2.as<uint32_t>(), R.Np, s));
                if (g_opts.sparsity != 0) {
                    TRY(R.occ.ensure((size_t)(Mt * Kt), "tile occupancy"));
                    LAUNCH(launch_tile_occupancy(R.at2.as<uint32_t>(), R.Np, R.Np, R.occ.as<uint8_t>(), s));
                    TRY(build_tile_lists(R, s));
                }
            } else {
                LAUNCH(launch_make_at2(R.a_src, R.a_ld, N, N, R.at2.as<uint32_t>(), R.Np, R.Np, R.flag.as<int>(), s));
            }
            R.has_at2 = true;
            R.sparse = g_opts.sparsity != 0;
            R.issued_per_product = R.sparse ? R.issued_tiles : (double)R.Np * R.Np * (double)R.ld;
        }
    }
    if (!R.has_at2) R.at2.release();

    tr.mark(R.spmm ? "kernel choice: spmm" : "kernel choice: tiles");
    // power store: a ring of device slots (allocated on first use, kept across calls).  The
    // slot count is decided once per (slot size, budget, max_k): cudaMemGetInfo can take
    // milliseconds when the driver has deferred work, so it is not called on every run.
    const std::tuple<size_t, int64_t, int, bool> ring_key{R.slot_bytes(), g_opts.budget, max_k, cap != nullptr};
    if (R.ring.empty() || ring_key != R.ring_key) {
        size_t freeb = 0, totalb = 0;
        CUDA_TRY(cudaMemGetInfo(&freeb, &totalb));
        size_t cached = 0;
        for (auto &b : R.ring) cached += b.bytes;
        const double avail = 0.90 * (double)(freeb + cached);
        const double cap_bytes = std::max((double)kDefaultRingBytes, 4.0 * (double)R.slot_bytes());
        int64_t budget = g_opts.budget > 0 ? g_opts.budget : (int64_t)std::min(avail, cap_bytes);
        int64_t slots = budget / (int64_t)R.slot_bytes();
        // an explicit budget also covers the two recompute buffers of an evicted partner
        if (g_opts.budget > 0) slots -= 2;
        // a batched run (small N) needs the whole batch resident (one more slot if the run can
        // go past the first batch); the batch size depends on N only, so every rank of a
        // sharded run issues the same collective calls
        const int64_t bsz = (N <= kBatchMaxN && !cap) ? std::min(kBatch, max_k) : 1;
        const int64_t need = bsz + (max_k > bsz ? 1 : 0) > 2 ? bsz + (max_k > bsz ? 1 : 0) : 2;
        slots = std::min<int64_t>(slots, std::max<int64_t>(max_k, need));
        if (slots < need)
            return fail(MP_ERR_RESOURCE, "power store needs at least %lld slots of %zu bytes (budget %lld bytes)",
                        (long long)need, R.slot_bytes(), (long long)budget);
        R.ring.resize((size_t)slots);
        R.ring_key = ring_key;
    }
    R.slot_power.assign(R.ring.size(), 0);
    tr.mark("power store");
    // per-power statistics: SUM fields {H, inf count} for k = 0..max_k, then MIN fields
    // {diag min, first finite entry}, so a batch of powers reduces with one call of each
    const size_t nst = (size_t)(max_k + 1) * 2;
    TRY(R.stats.ensure(nst * 2 * 8, "per-power statistics"));
    TRY(R.flag.ensure(16, "compare flag"));
    int64_t *st_sum = R.stats.as<int64_t>(), *st_min = st_sum + nst;
    {
        std::vector<int64_t> init(nst * 2, 0);
        for (size_t q = nst; q < init.size(); q += 2) {
            init[q] = 0xFFFF;
            init[q + 1] = INT64_MAX;
        }
        COPY(R.stats.p, init.data(), init.size() * 8, cudaMemcpyHostToDevice, s);
    }
    // the fingerprint on the tensor cores for symmetric runs
    R.fptc = R.sym && fp_tc_on() && R.w > 0;
    if (R.fptc) {
        TRY(R.tcs.ensure(nst * 8, "tensor-core fingerprints"));
        CUDA_TRY(cudaMemsetAsync(R.tcs.p, 0, nst * 8, s));
        TRY(R.wfrag.ensure((size_t)(R.ld / 32) * 32 * 16, "fingerprint weight fragments"));
        LAUNCH(launch_fp_tc_weights(R.dgcol.as<int32_t>(), R.dsig.as<int32_t>(), R.w, R.ld, R.wfrag.as<uint4>(), s));
    }
    unsigned long long *tcs = R.fptc ? R.tcs.as<unsigned long long>() : nullptr;
    // Batch of powers between host synchronisations: products of small matrices take
    // microseconds, so up to kBatch of them are enqueued back to back and their statistics
    // read with one copy; powers computed past the first repeat are discarded.  The batch
    // depends only on N, so every rank of a sharded run makes the same collective calls.
    const int B = (N <= kBatchMaxN && !cap) ? std::min(kBatch, max_k) : 1; // ring >= B + 1 (above)
    // events: [0, 2(max_k+1)) product start/stop per power, then stats start, stats stop
    if ((int)R.events.size() < 5 * (max_k + 1)) {
        for (auto ev : R.events) cudaEventDestroy(ev);
        R.events.assign((size_t)5 * (max_k + 1), nullptr);
        for (auto &ev : R.events) CUDA_TRY(cudaEventCreate(&ev));
    }

    std::vector<mp_power_stats> hs((size_t)max_k + 1);
    const uint64_t S = mp_fingerprint_unit(N); // O(N) on the host
    double prod_ms = 0.0, stats_ms = 0.0, spmm_ms = 0.0;
    int64_t launches = 0;
    cudaEvent_t ev_setup;
    CUDA_TRY(cudaEventCreate(&ev_setup));
    CUDA_TRY(cudaEventRecord(ev_setup, s));
    tr.mark("statistics init");

    mp_periodic_result res;
    std::memset(&res, 0, sizeof(res));
    const uint16_t *prev = nullptr;
    std::vector<const uint16_t *> buf((size_t)max_k + 1, nullptr);
    std::vector<int64_t> hsum(nst), hmin(nst);
    bool found = false;
    // Lookahead (large N, one rank, no observer): product k+1 runs on the library stream while
    // the statistics of power k run on a second stream and the host searches for a repeat, so
    // the statistics overlap the next product and the host round trip is hidden.  A power past
    // the first repeat is computed and discarded (one product per run).
    // (measured: n = 10 10.7 -> 9.8 ms, n = 11 36.4 -> 33.3 ms; at n = 12 the statistics slow the
    // memory-bound product they overlap by more than the hidden round trip: 177.6 vs 179.6 ms)
    const bool lookahead = B == 1 && !cap && !g_dist.fn && !g_obs.fn && max_k >= 2 && R.ring.size() >= 3 &&
                           (N < kLookaheadMaxN || lookahead_forced()) && lookahead_on();
    if (lookahead) {
        cudaStream_t s2 = st->stream2;
        if (!s2) {
            CUDA_TRY(cudaStreamCreateWithFlags(&st->stream2, cudaStreamNonBlocking));
            s2 = st->stream2;
        }
        if (!R.hstats || R.hstats_n < nst * 2) {
            if (R.hstats) cudaFreeHost(R.hstats);
            R.hstats = nullptr;
            CUDA_TRY(cudaMallocHost((void **)&R.hstats, nst * 2 * 8));
            R.hstats_n = nst * 2;
        }
        if ((int)R.events_la.size() < 2 * (max_k + 1) + 2) {
            for (auto ev : R.events_la) cudaEventDestroy(ev);
            R.events_la.assign((size_t)2 * (max_k + 1) + 2, nullptr);
            for (auto &ev : R.events_la) CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        }
        int64_t *hsum_p = R.hstats, *hmin_p = R.hstats + nst;
        cudaEvent_t *prod_done = R.events_la.data(), *stats_done = R.events_la.data() + (max_k + 1);
        cudaEvent_t join = R.events_la[2 * (max_k + 1)], start2 = R.events_la[2 * (max_k + 1) + 1];
        CUDA_TRY(cudaEventRecord(start2, s)); // the second stream starts after the setup
        CUDA_TRY(cudaStreamWaitEvent(s2, start2, 0));
        // enqueue power k: the product (or X_1) on s, its statistics and their copy to the host
        // on s2 once the product is done
        auto issue = [&](int k) -> mp_status {
            const size_t q = (size_t)(k % (int)R.ring.size());
            TRY(R.ring[q].ensure(R.slot_bytes(), "power store slot"));
            uint16_t *dst = R.ring[q].as<uint16_t>();
            R.slot_power[q] = k;
            buf[(size_t)k] = dst;
            if (k == 1) {
                TRY(make_power1(R, dst, s));
            }
            if (k >= 2) {
                CUDA_TRY(cudaEventRecord(R.events[2 * k], s));
                TRY(product(R, buf[(size_t)k - 1], dst, s, R.events[4 * (max_k + 1) + k]));
                CUDA_TRY(cudaEventRecord(R.events[2 * k + 1], s));
                ++launches;
            }
            CUDA_TRY(cudaEventRecord(prod_done[k], s));
            CUDA_TRY(cudaStreamWaitEvent(s2, prod_done[k], 0));
            CUDA_TRY(cudaEventRecord(R.events[2 * (max_k + 1) + k], s2));
            if (R.sym) {
                if (tcs)
                    LAUNCH(launch_fp_tc(dst, R.ld, N, R.w, R.wfrag.as<uint4>(), R.drw.as<uint64_t>(),
                                        R.drw.as<uint64_t>() + N, tcs + 2 * k, s2, k >= 2 ? tcs + 2 * (k - 1) : nullptr));
                LAUNCH(launch_stats_sym(dst, R.ld, N, R.dgcol.as<int32_t>(), R.dsig.as<int32_t>(), R.drw.as<uint64_t>(),
                                        R.drw.as<uint64_t>() + N, R.w,
                                        reinterpret_cast<unsigned long long *>(st_sum + 2 * k),
                                        reinterpret_cast<unsigned long long *>(st_min + 2 * k), s2,
                                        tcs ? tcs + 2 * k : nullptr));
            }
            else
                LAUNCH(launch_stats(dst, R.ld, N, R.c0, R.w, reinterpret_cast<unsigned long long *>(st_sum + 2 * k),
                                    reinterpret_cast<unsigned long long *>(st_min + 2 * k), s2));
            CUDA_TRY(cudaEventRecord(R.events[3 * (max_k + 1) + k], s2));
            COPY(hsum_p + 2 * k, st_sum + 2 * k, 16, cudaMemcpyDeviceToHost, s2);
            COPY(hmin_p + 2 * k, st_min + 2 * k, 16, cudaMemcpyDeviceToHost, s2);
            CUDA_TRY(cudaEventRecord(stats_done[k], s2));
            return MP_OK;
        };
        TRY(issue(1));
        int k_issued = 1;
        for (int k = 1; k <= max_k && !found; ++k) {
            if (k + 1 <= max_k) {
                TRY(issue(k + 1));
                k_issued = k + 1;
            }
            CUDA_TRY(cudaEventSynchronize(stats_done[k]));
            tr.mark("power + statistics", k);
            mp_power_stats &cs = hs[(size_t)k];
            cs.fingerprint = hsum_p[2 * k];
            cs.inf_count = hsum_p[2 * k + 1];
            cs.diag_min = hmin_p[2 * k];
            cs.ref = hmin_p[2 * k + 1];
            res.diag_min[k] = (uint16_t)std::min<int64_t>(cs.diag_min, 0xFFFF);
            res.fingerprint[k] = (uint64_t)cs.fingerprint;
            if (!res.dense_from && cs.inf_count == 0) res.dense_from = k;
            const uint16_t *cur = buf[(size_t)k];
            // a5: forward first-repeat search, j = k-1 down to 1; the exact compare runs on s2
            for (int j = k - 1; j >= 1 && !found; --j) {
                int32_t c = 0;
                if (!mp_repeat_candidate(&cs, &hs[(size_t)j], S, &c)) continue;
                const uint16_t *Z = nullptr;
                bool in_ring = false;
                for (size_t q = 0; q < R.ring.size(); ++q)
                    if (R.slot_power[q] == j) in_ring = true;
                if (!in_ring) CUDA_TRY(cudaStreamSynchronize(s)); // the recompute runs on s
                TRY(power_buffer(R, j, &Z, in_ring ? s2 : s));
                if (!in_ring) CUDA_TRY(cudaStreamSynchronize(s));
                int64_t *fl = R.flag.as<int64_t>();
                CUDA_TRY(cudaMemsetAsync(fl, 0, 8, s2));
                LAUNCH(launch_compare(cur, Z, R.ld, N, R.w, c, reinterpret_cast<unsigned long long *>(fl), s2));
                int64_t bad = -1;
                COPY(&bad, fl, 8, cudaMemcpyDeviceToHost, s2);
                CUDA_TRY(cudaStreamSynchronize(s2));
                if (bad == 0) {
                    found = true;
                    res.mu = j;
                    res.lambda = k - j;
                    res.offset = c;
                    res.k_last = k;
                }
            }
        }
        CUDA_TRY(cudaEventRecord(join, s2)); // the library stream waits for the second one
        CUDA_TRY(cudaStreamWaitEvent(s, join, 0));
        CUDA_TRY(cudaStreamSynchronize(s));
        for (int k = 2; k <= k_issued; ++k) { // timings (the discarded lookahead power included)
            float ms = 0.f;
            CUDA_TRY(cudaEventElapsedTime(&ms, R.events[2 * k], R.events[2 * k + 1]));
            prod_ms += ms;
            if (R.spmm) {
                CUDA_TRY(cudaEventElapsedTime(&ms, R.events[2 * k], R.events[4 * (max_k + 1) + k]));
                spmm_ms += ms;
            }
            CUDA_TRY(cudaEventElapsedTime(&ms, R.events[2 * (max_k + 1) + k], R.events[3 * (max_k + 1) + k]));
            stats_ms += ms;
        }
    }
    for (int kb = 1; kb <= max_k && !found && !lookahead; kb += B) {
        const int ke = std::min(max_k, kb + B - 1);
        for (int k = kb; k <= ke; ++k) {
            const size_t q = (size_t)(k % (int)R.ring.size());
            TRY(R.ring[q].ensure(R.slot_bytes(), "power store slot"));
            uint16_t *dst = R.ring[q].as<uint16_t>();
            R.slot_power[q] = k;
            buf[(size_t)k] = dst;
            if (k == 1) {
                TRY(make_power1(R, dst, s)); // X_1 = A[:, shard]
            } else {
                CUDA_TRY(cudaEventRecord(R.events[2 * k], s));
                TRY(product(R, prev, dst, s, R.events[4 * (max_k + 1) + k])); // A^k = A (x) A^{k-1}
                CUDA_TRY(cudaEventRecord(R.events[2 * k + 1], s));
                ++launches;
            }
            if (k >= 2) CUDA_TRY(cudaEventRecord(R.events[2 * (max_k + 1) + k], s)); // stats start
            if (R.sym) {
                if (tcs)
                    LAUNCH(launch_fp_tc(dst, R.ld, N, R.w, R.wfrag.as<uint4>(), R.drw.as<uint64_t>(),
                                        R.drw.as<uint64_t>() + N, tcs + 2 * k, s, k >= 2 ? tcs + 2 * (k - 1) : nullptr));
                LAUNCH(launch_stats_sym(dst, R.ld, N, R.dgcol.as<int32_t>(), R.dsig.as<int32_t>(),
                                        R.drw.as<uint64_t>(), R.drw.as<uint64_t>() + N, R.w,
                                        reinterpret_cast<unsigned long long *>(st_sum + 2 * k),
                                        reinterpret_cast<unsigned long long *>(st_min + 2 * k), s,
                                        tcs ? tcs + 2 * k : nullptr));
            }
            else
                LAUNCH(launch_stats(dst, R.ld, N, R.c0, R.w, reinterpret_cast<unsigned long long *>(st_sum + 2 * k),
                                    reinterpret_cast<unsigned long long *>(st_min + 2 * k), s));
            if (k >= 2) CUDA_TRY(cudaEventRecord(R.events[3 * (max_k + 1) + k], s)); // stats end
            prev = dst;
        }
        const int nb = ke - kb + 1;
        TRY(allreduce(0, st_sum + 2 * kb, 2 * nb, s)); // SUM: fingerprint, inf count
        TRY(allreduce(1, st_min + 2 * kb, 2 * nb, s)); // MIN: diagonal minimum, first finite entry
        COPY(hsum.data() + 2 * kb, st_sum + 2 * kb, (size_t)nb * 16, cudaMemcpyDeviceToHost, s);
        COPY(hmin.data() + 2 * kb, st_min + 2 * kb, (size_t)nb * 16, cudaMemcpyDeviceToHost, s);
        CUDA_TRY(cudaStreamSynchronize(s));
        tr.mark("powers + statistics", ke);

        for (int k = kb; k <= ke && !found; ++k) {
            if (k >= 2) {
                float ms = 0.f;
                CUDA_TRY(cudaEventElapsedTime(&ms, R.events[2 * k], R.events[2 * k + 1]));
                prod_ms += ms;
                if (R.spmm) {
                    CUDA_TRY(cudaEventElapsedTime(&ms, R.events[2 * k], R.events[4 * (max_k + 1) + k]));
                    spmm_ms += ms;
                }
                CUDA_TRY(cudaEventElapsedTime(&ms, R.events[2 * (max_k + 1) + k], R.events[3 * (max_k + 1) + k]));
                stats_ms += ms;
            }
            mp_power_stats &cs = hs[(size_t)k];
            cs.fingerprint = hsum[2 * k];
            cs.inf_count = hsum[2 * k + 1];
            cs.diag_min = hmin[2 * k];
            cs.ref = hmin[2 * k + 1];
            res.diag_min[k] = (uint16_t)std::min<int64_t>(cs.diag_min, 0xFFFF);
            res.fingerprint[k] = (uint64_t)cs.fingerprint;
            if (!res.dense_from && cs.inf_count == 0) res.dense_from = k;
            const uint16_t *cur = buf[(size_t)k];
            if (g_obs.fn && !cap) TRY(observe(R, cur, k, s));

            if (cap) {
                DBuf rowbuf;
                TRY(rowbuf.alloc((size_t)N * 4, "captured row"));
                std::vector<uint16_t> h2((size_t)R.w * 2);
                for (int r = 0; r < cap->nrows; ++r) {
                    uint16_t *o = cap->out + ((size_t)(k - 1) * cap->nrows + r) * N;
                    const int64_t row = cap->rows[r];
                    if (!R.sym) {
                        LAUNCH(launch_decode(cur + row * R.ld, R.ld, 1, N, rowbuf.as<uint16_t>(), N, s));
                        CUDA_TRY(cudaMemcpyAsync(o, rowbuf.p, (size_t)N * 2, cudaMemcpyDeviceToHost, s));
                        CUDA_TRY(cudaStreamSynchronize(s));
                        continue;
                    }
                    // full row r from the domain columns: X_rj = X_(r, j) if j <= sigma j,
                    // else X_(sigma r, sigma j)
                    uint16_t *rb = rowbuf.as<uint16_t>();
                    LAUNCH(launch_decode(cur + row * R.ld, R.ld, 1, R.w, rb, R.w, s));
                    LAUNCH(launch_decode(cur + (int64_t)R.sigma[row] * R.ld, R.ld, 1, R.w, rb + R.w, R.w, s));
                    CUDA_TRY(cudaMemcpyAsync(h2.data(), rb, (size_t)R.w * 4, cudaMemcpyDeviceToHost, s));
                    CUDA_TRY(cudaStreamSynchronize(s));
                    for (int64_t j = 0; j < N; ++j) {
                        const int32_t sj = R.sigma[j];
                        o[j] = j <= sj ? h2[(size_t)R.loc[j]] : h2[(size_t)(R.w + R.loc[sj])];
                    }
                }
                if (k == max_k) found = true;
                continue;
            }

            // a5: forward first-repeat search, j = k-1 down to 1
            for (int j = k - 1; j >= 1 && !found; --j) {
                int32_t c = 0;
                if (!mp_repeat_candidate(&cs, &hs[(size_t)j], S, &c)) continue;
                const uint16_t *Z = nullptr;
                TRY(power_buffer(R, j, &Z, s));
                int64_t *fl = R.flag.as<int64_t>();
                CUDA_TRY(cudaMemsetAsync(fl, 0, 8, s));
                LAUNCH(launch_compare(cur, Z, R.ld, N, R.w, c, reinterpret_cast<unsigned long long *>(fl), s));
                TRY(allreduce(0, fl, 1, s));
                int64_t bad = -1;
                COPY(&bad, fl, 8, cudaMemcpyDeviceToHost, s);
                CUDA_TRY(cudaStreamSynchronize(s));
                if (bad == 0) {
                    found = true;
                    res.mu = j;
                    res.lambda = k - j;
                    res.offset = c;
                    res.k_last = k;
                }
            }
        }
        for (int k = std::max(2, kb); k <= ke && found && !cap; ++k) // discarded powers still ran
            if (k > res.k_last) {
                float ms = 0.f;
                CUDA_TRY(cudaEventElapsedTime(&ms, R.events[2 * k], R.events[2 * k + 1]));
                prod_ms += ms;
                if (R.spmm) {
                    CUDA_TRY(cudaEventElapsedTime(&ms, R.events[2 * k], R.events[4 * (max_k + 1) + k]));
                    spmm_ms += ms;
                }
            }
    }
    CUDA_TRY(cudaEventRecord(ev_all1, s));
    CUDA_TRY(cudaEventSynchronize(ev_all1));
    float all_ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&all_ms, ev_all0, ev_all1));
    cudaEventDestroy(ev_all1);

    // dense-equivalent steps count the products up to the first repeat (useful work); the
    // launches and their time include any product of the batch computed past it
    const int64_t useful = found && !cap ? (int64_t)res.k_last - 1 : launches;
    g_prof.product_ms = prod_ms;
    g_prof.stats_ms = stats_ms;
    g_prof.product_launches = launches;
    g_prof.dense_steps = (double)useful * (double)N * (double)N * (double)R.cols_rep;
    g_prof.issued_steps = (double)launches * R.issued_per_product;
    g_prof.total_ms = all_ms;
    {
        float sms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&sms, ev_all0, ev_setup));
        g_prof.setup_ms = sms;
        cudaEventDestroy(ev_setup);
        cudaEventDestroy(ev_all0);
    }
    g_prof.h2d_bytes = g_h2d.load() - h2d0;
    g_prof.d2h_bytes = g_d2h.load() - d2h0;
    g_prof.kernel = R.spmm ? 2 : (R.sparse ? 1 : 0);
    g_prof.spmm_cols = R.spmm ? R.sp.cols : 0;
    g_prof.local_cols = R.w;
    g_prof.ld = R.ld;
    g_prof.spmm_ms = R.spmm ? spmm_ms : prod_ms;
    g_prof.row_levels = R.spmm && R.dag_n ? R.rdag.levels : 0;
    g_prof.row_parents = R.spmm && R.dag_n ? R.rdag.parents : 0;
    g_prof.fold_bytes = R.spmm && R.dag_n ? (double)R.rdag.fold_rows * (double)R.ld * 2.0 : 0.0;

    if (!found) return fail(MP_ERR_NOT_PERIODIC, "no repeat A^k = c (x) A^j with k <= %d", max_k);
    *out = res;
    return MP_OK;
}

} // namespace

// =======================================================================================
// Public ABI
// =======================================================================================
extern "C" {

mp_status mp_count_words(int n, int64_t *N_out)
{
    if (!N_out || n < 2 || n > MP_MAX_N)
        return fail(MP_ERR_DOMAIN, "mp_count_words: n = %d outside [2, %d]", n, MP_MAX_N);
    *N_out = count_words(n);
    return MP_OK;
}

mp_status build_transition_matrix_into(int n, uint16_t *A, int64_t N)
{
    if (!A || n < 2 || n > MP_MAX_N)
        return fail(MP_ERR_DOMAIN, "build_transition_matrix: n = %d outside [2, %d] or NULL buffer", n, MP_MAX_N);
    const std::vector<WordMask> words = enumerate_words(n);
    if ((int64_t)words.size() != N)
        return fail(MP_ERR_DOMAIN, "build_transition_matrix: N = %lld but |C_%d| = %zu", (long long)N, n,
                    words.size());
    fill_transition_matrix(words, n, A, host_threads());
    return MP_OK;
}

mp_status build_transition_matrix(int n, uint16_t **A_out, int64_t *N_out)
{
    if (!A_out || !N_out || n < 2 || n > MP_MAX_N)
        return fail(MP_ERR_DOMAIN, "build_transition_matrix: n = %d outside [2, %d] or NULL output", n, MP_MAX_N);
    const int64_t N = count_words(n);
    const size_t bytes = (size_t)N * (size_t)N * 2;
    uint16_t *A = (uint16_t *)std::malloc(bytes);
    if (!A) return fail(MP_ERR_RESOURCE, "host allocation of %zu bytes for A(D_%d) failed", bytes, n);
    mp_status s = build_transition_matrix_into(n, A, N);
    if (s != MP_OK) {
        std::free(A);
        return s;
    }
    *A_out = A;
    *N_out = N;
    return MP_OK;
}

void mp_free(void *p) { std::free(p); }

mp_status minplus_mul(const uint16_t *A, const uint16_t *B, uint16_t *C, int64_t M, int64_t K, int64_t N)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!A || !B || !C || M <= 0 || K <= 0 || N <= 0)
        return fail(MP_ERR_DOMAIN, "minplus_mul: NULL pointer or non-positive dimension (M=%lld K=%lld N=%lld)",
                    (long long)M, (long long)K, (long long)N);
    if (overlaps(C, (size_t)M * N * 2, A, (size_t)M * K * 2) || overlaps(C, (size_t)M * N * 2, B, (size_t)K * N * 2))
        return fail(MP_ERR_DOMAIN, "minplus_mul: C overlaps A or B");
    int dev = 0;
    DevState *st = nullptr;
    TRY(current_device(&dev, &st));
    cudaStream_t s = st->stream;
    TRY(st->stage_a.ensure((size_t)M * K * 2, "A staging"));
    TRY(st->stage_b.ensure((size_t)K * N * 2, "B staging"));
    TRY(st->stage_c.ensure((size_t)M * N * 2, "C staging"));
    COPY(st->stage_a.p, A, (size_t)M * K * 2, cudaMemcpyHostToDevice, s);
    COPY(st->stage_b.p, B, (size_t)K * N * 2, cudaMemcpyHostToDevice, s);
    if (sharded_products())
        TRY(mul_sharded(*st, st->stage_a.as<uint16_t>(), st->stage_b.as<uint16_t>(), N, st->stage_c.as<uint16_t>(),
                        M, K, N, s));
    else
        TRY(mul_device_impl(*st, st->stage_a.as<uint16_t>(), K, st->stage_b.as<uint16_t>(), N,
                            st->stage_c.as<uint16_t>(), N, M, K, N, s));
    COPY(C, st->stage_c.p, (size_t)M * N * 2, cudaMemcpyDeviceToHost, s);
    CUDA_TRY(cudaStreamSynchronize(s));
    return MP_OK;
}

mp_status minplus_mul_device(const uint16_t *dA, int64_t lda, const uint16_t *dB, int64_t ldb, uint16_t *dC,
                             int64_t ldc, int64_t M, int64_t K, int64_t N, void *stream)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!dA || !dB || !dC || M <= 0 || K <= 0 || N <= 0 || lda < K || ldb < N || ldc < N)
        return fail(MP_ERR_DOMAIN, "minplus_mul_device: NULL pointer, non-positive dimension or ld < cols");
    if (overlaps(dC, span_bytes(M, N, ldc), dA, span_bytes(M, K, lda)) ||
        overlaps(dC, span_bytes(M, N, ldc), dB, span_bytes(K, N, ldb)))
        return fail(MP_ERR_DOMAIN, "minplus_mul_device: C overlaps A or B");
    int dev = 0;
    DevState *st = nullptr;
    TRY(current_device(&dev, &st));
    return mul_device_impl(*st, dA, lda, dB, ldb, dC, ldc, M, K, N, (cudaStream_t)stream);
}

mp_status minplus_mul_strided_batched_device(const uint16_t *dA, int64_t lda, int64_t strideA, const uint16_t *dB,
                                             int64_t ldb, int64_t strideB, uint16_t *dC, int64_t ldc, int64_t strideC,
                                             int64_t M, int64_t K, int64_t N, int64_t batch, void *stream)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!dA || !dB || !dC || M <= 0 || K <= 0 || N <= 0 || batch <= 0 || lda < K || ldb < N || ldc < N ||
        strideA < 0 || strideB < 0 || strideC < 0)
        return fail(MP_ERR_DOMAIN, "minplus_mul_strided_batched_device: NULL pointer, non-positive dimension, "
                                   "ld < cols or negative stride");
    const size_t cspan = span_bytes(M, N, ldc);
    if (batch > 1 && (size_t)strideC * 2 < cspan)
        return fail(MP_ERR_DOMAIN, "minplus_mul_strided_batched_device: the C matrices overlap (strideC too small)");
    const size_t ca = (size_t)(batch - 1) * (size_t)strideC * 2 + cspan;
    if (overlaps(dC, ca, dA, (size_t)(batch - 1) * (size_t)strideA * 2 + span_bytes(M, K, lda)) ||
        overlaps(dC, ca, dB, (size_t)(batch - 1) * (size_t)strideB * 2 + span_bytes(K, N, ldb)))
        return fail(MP_ERR_DOMAIN, "minplus_mul_strided_batched_device: C overlaps A or B");
    int dev = 0;
    DevState *st = nullptr;
    TRY(current_device(&dev, &st));
    return mul_device_impl(*st, dA, lda, strideA, dB, ldb, strideB, dC, ldc, strideC, M, K, N, batch,
                           (cudaStream_t)stream);
}

mp_status minplus_closure(const uint16_t *W, int64_t N, uint16_t *D, int32_t *squarings_out)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!W || !D || N <= 0) return fail(MP_ERR_DOMAIN, "minplus_closure: NULL pointer or N <= 0");
    if (overlaps(D, (size_t)N * N * 2, W, (size_t)N * N * 2)) return fail(MP_ERR_DOMAIN, "minplus_closure: D overlaps W");
    int dev = 0;
    DevState *st = nullptr;
    TRY(current_device(&dev, &st));
    cudaStream_t s = st->stream;
    TRY(st->stage_a.ensure((size_t)N * N * 2, "closure buffer"));
    TRY(st->stage_b.ensure((size_t)N * N * 2, "closure buffer"));
    uint16_t *X = st->stage_a.as<uint16_t>(), *Y = st->stage_b.as<uint16_t>();
    COPY(X, W, (size_t)N * N * 2, cudaMemcpyHostToDevice, s);
    LAUNCH(launch_set_diag_zero(X, N, N, s)); // I (+) W: every vertex reaches itself at cost 0
    int32_t t = 0;
    for (int64_t reach = 1; reach < N - 1; reach *= 2, ++t) { // (I + W)^(2^t) covers paths of 2^t arcs
        if (sharded_products()) // X is replicated: each rank squares its column block, then all-gather
            TRY(mul_sharded(*st, X, X, N, Y, N, N, N, s));
        else
            TRY(mul_device_impl(*st, X, N, X, N, Y, N, N, N, N, s));
        std::swap(X, Y);
    }
    COPY(D, X, (size_t)N * N * 2, cudaMemcpyDeviceToHost, s);
    CUDA_TRY(cudaStreamSynchronize(s));
    if (squarings_out) *squarings_out = t;
    return MP_OK;
}

mp_status minplus_power_until_periodic(const uint16_t *A, int64_t N, int max_k, mp_periodic_result *out)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!A || !out || N <= 0 || max_k < 2 || max_k > MP_MAX_K)
        return fail(MP_ERR_DOMAIN, "minplus_power_until_periodic: NULL pointer, N <= 0 or max_k outside [2, %d]",
                    MP_MAX_K);
    ASource src;
    src.host = A;
    return run_powers(src, N, max_k, out);
}

mp_status minplus_power_until_periodic_device(const uint16_t *dA, int64_t lda, int64_t N, int max_k,
                                              mp_periodic_result *out)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!dA || !out || N <= 0 || lda < N || max_k < 2 || max_k > MP_MAX_K)
        return fail(MP_ERR_DOMAIN,
                    "minplus_power_until_periodic_device: NULL pointer, N <= 0, lda < N or max_k outside [2, %d]",
                    MP_MAX_K);
    ASource src;
    src.dev = dA;
    src.lda = lda;
    return run_powers(src, N, max_k, out);
}

mp_status minplus_power_rows(const uint16_t *A, int64_t N, int kmax, const int64_t *rows, int nrows, uint16_t *out)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!A || !rows || !out || N <= 0 || kmax < 1 || kmax > MP_MAX_K || nrows <= 0)
        return fail(MP_ERR_DOMAIN, "minplus_power_rows: invalid arguments");
    for (int r = 0; r < nrows; ++r)
        if (rows[r] < 0 || rows[r] >= N) return fail(MP_ERR_DOMAIN, "minplus_power_rows: row %lld outside [0, N)",
                                                     (long long)rows[r]);
    ASource src;
    src.host = A;
    Capture cap;
    cap.rows = rows;
    cap.nrows = nrows;
    cap.out = out;
    mp_periodic_result res;
    const Dist saved = g_dist;
    g_dist = Dist();
    mp_status st = run_powers(src, N, kmax, &res, &cap);
    g_dist = saved;
    return st;
}

mp_status mp_gamma2_readoff(const mp_periodic_result *r, int64_t m, int64_t *g)
{
    if (!r || !g || m < 3 || r->lambda <= 0 || r->k_last <= 0)
        return fail(MP_ERR_DOMAIN, "mp_gamma2_readoff: m = %lld < 3 or invalid result", (long long)m);
    if (m <= r->k_last) {
        *g = r->diag_min[m];
        return MP_OK;
    }
    // Theorem 3: gamma(m) = gamma(m - t*lambda) + t*b, m - t*lambda in (mu, k_last]
    const int64_t t = (m - r->k_last + r->lambda - 1) / r->lambda;
    *g = (int64_t)r->diag_min[m - t * r->lambda] + t * (int64_t)r->offset;
    return MP_OK;
}

mp_status mp_gamma2_formula(const mp_periodic_result *r, mp_formula *out)
{
    if (!r || !out || r->lambda <= 0 || r->lambda > MP_MAX_K || r->mu < 1 || r->k_last != r->mu + r->lambda)
        return fail(MP_ERR_DOMAIN, "mp_gamma2_formula: NULL or invalid periodic result");
    mp_formula f;
    std::memset(&f, 0, sizeof(f));
    f.a = r->lambda;
    f.b = r->offset;
    f.n0 = r->mu;
    f.r0_k50 = (50 >= r->mu + r->lambda) ? 50 - r->lambda : -1;
    auto ceil_div = [](int64_t x, int64_t y) { return (x + y - 1) / y; };
    // boundary values gamma_2(m), n0 <= m < n0 + a (Algorithm 5) fix alpha per residue
    for (int64_t m = r->mu; m < r->mu + r->lambda; ++m) {
        if (m < 3) continue; // gamma_2 undefined below 3 (G17): use m + a instead
        f.alpha[m % f.a] = (int32_t)(r->diag_min[m] - ceil_div((int64_t)f.b * m, f.a));
    }
    for (int64_t m = r->mu; m < 3; ++m) { // n0 < 3: take the residue from m + a (Lemma 1)
        const int64_t mm = m + f.a;
        f.alpha[m % f.a] = (int32_t)(r->diag_min[mm] - ceil_div((int64_t)f.b * mm, f.a));
    }
    for (int64_t m = 3; m < r->mu && f.n_exceptions < MP_MAX_K; ++m) {
        const int64_t formula = ceil_div((int64_t)f.b * m, f.a) + f.alpha[m % f.a];
        if ((int64_t)r->diag_min[m] != formula) {
            f.exception_m[f.n_exceptions] = m;
            f.exception_gamma2[f.n_exceptions] = r->diag_min[m];
            ++f.n_exceptions;
        }
    }
    *out = f;
    return MP_OK;
}

mp_status mp_gamma2_record(int n, mp_periodic_result *out)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!out || n < 2 || n > MP_MAX_N)
        return fail(MP_ERR_DOMAIN, "mp_gamma2_record: n = %d outside [2, %d] or NULL", n, MP_MAX_N);
    const auto key = std::make_tuple(n, g_dist.world, g_dist.rank);
    auto it = g_cache.find(key);
    if (it == g_cache.end()) {
        mp_periodic_result r;
        ASource src;
        src.n = n;
        TRY(run_powers(src, count_words(n), 64, &r));
        it = g_cache.emplace(key, r).first;
    }
    *out = it->second;
    return MP_OK;
}

mp_status gamma2_cylinder(int n, int64_t m, int64_t *gamma2_out)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!gamma2_out || n < 2 || n > MP_MAX_N || m < 3)
        return fail(MP_ERR_DOMAIN, "gamma2_cylinder: n = %d outside [2, %d] or m = %lld < 3", n, MP_MAX_N,
                    (long long)m);
    mp_periodic_result r;
    TRY(mp_gamma2_record(n, &r));
    return mp_gamma2_readoff(&r, m, gamma2_out);
}

mp_status mp_dist_set(int rank, int world, mp_allreduce_fn fn, void *ctx)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (fn == nullptr) {
        g_dist = Dist();
        return MP_OK;
    }
    const mp_allgather_fn keep = g_dist.gather;
    void *keep_ctx = g_dist.gctx;
    if (world < 1 || rank < 0 || rank >= world)
        return fail(MP_ERR_DOMAIN, "mp_dist_set: rank %d / world %d invalid", rank, world);
    g_dist.rank = rank;
    g_dist.world = world;
    g_dist.fn = fn;
    g_dist.ctx = ctx;
    g_dist.gather = keep;
    g_dist.gctx = keep_ctx;
    return MP_OK;
}

mp_status mp_dist_set_allgather(mp_allgather_fn fn, void *ctx)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    g_dist.gather = fn;
    g_dist.gctx = fn ? ctx : nullptr;
    return MP_OK;
}

mp_status mp_shard_range(int64_t N, int world, int rank, int64_t *c0, int64_t *c1)
{
    if (!c0 || !c1 || N <= 0 || world < 1 || rank < 0 || rank >= world)
        return fail(MP_ERR_DOMAIN, "mp_shard_range: invalid arguments");
    const int64_t w = round_up((N + world - 1) / world, 8);
    *c0 = std::min<int64_t>(N, (int64_t)rank * w);
    *c1 = std::min<int64_t>(N, *c0 + w);
    return MP_OK;
}

mp_status mp_column_plan(int64_t N, int64_t w, int64_t *ld, int32_t *main_cols, int32_t *tail_cols)
{
    if (!ld || !main_cols || !tail_cols || N <= 0 || w < 0)
        return fail(MP_ERR_DOMAIN, "mp_column_plan: invalid arguments");
    const SpmmPlan P = spmm_plan(pad_rows(N), w);
    *ld = P.ld;
    *main_cols = P.main_cols;
    int32_t tail = 0;
    for (int g = 0; g < P.nseg; ++g)
        if (P.seg[g].cols != P.main_cols) tail += (int32_t)P.seg[g].ncols;
    *tail_cols = tail;
    return MP_OK;
}

uint64_t mp_fingerprint_unit(int64_t N)
{
    // S(N) = sum over i, j < N of s(2i) s(2j+1) = (sum_i s(2i)) (sum_j s(2j+1))  (mod 2^64)
    uint64_t a = 0, b = 0;
    for (int64_t i = 0; i < N; ++i) {
        a += mix64(2 * (uint64_t)i);
        b += mix64(2 * (uint64_t)i + 1);
    }
    return a * b;
}

int mp_repeat_candidate(const mp_power_stats *sk, const mp_power_stats *sj, uint64_t S, int32_t *c_out)
{
    if (!sk || !sj) return 0;
    if (sk->inf_count != sj->inf_count) return 0;
    const bool allinf_k = sk->ref == INT64_MAX, allinf_j = sj->ref == INT64_MAX;
    if (allinf_k || allinf_j) {
        if (allinf_k != allinf_j) return 0;
        if (c_out) *c_out = 0;
        return 1;
    }
    if ((sk->ref >> 16) != (sj->ref >> 16)) return 0; // first finite entries at different places
    const int32_t c = (int32_t)(sk->ref & 0xFFFF) - (int32_t)(sj->ref & 0xFFFF);
    if (c_out) *c_out = c;
    if (sk->inf_count > 0) return 1; // +inf present: the linear hash is not shift-equivariant
    const uint64_t lhs = (uint64_t)sk->fingerprint - (uint64_t)sj->fingerprint;
    const uint64_t rhs = (uint64_t)(int64_t)c * S;
    return lhs == rhs ? 1 : 0;
}

const char *mp_last_error(void) { return t_err.c_str(); }

void mp_shutdown(void)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    g_cache.clear();
    for (auto &kv : g_dev) {
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(kv.first);
        kv.second.pr.reset();
        if (kv.second.scratch_ev) cudaEventDestroy(kv.second.scratch_ev);
        if (kv.second.stream2) cudaStreamDestroy(kv.second.stream2);
        kv.second.stream2 = nullptr;
        kv.second.scratch_ev = nullptr;
        if (kv.second.stream) cudaStreamDestroy(kv.second.stream);
        kv.second.stream = nullptr;
        cudaSetDevice(cur);
    }
    g_dev.clear();
}

const char *mp_version(void)
{
    return "minplus-b200 0.5 sm_100a: DPX VIADDMNMX.U16x2; 128x256x32 tile kernel (dense / block-sparse, 4-stage "
           "cp.async) and warp-specialised grouped SpMM (4-row groups, greedy row grouping; extras order under the "
           "reuse, bulk copies + mbarrier ring); column symmetry; row-inclusion reuse (SpMM on the extra entries + "
           "fold passes); u8 IMMA fingerprint; one-cluster small-N kernel";
}

int64_t mp_kernel_launches(void) { return g_launches.load(); }

mp_status mp_last_profile(mp_profile *out)
{
    if (!out) return fail(MP_ERR_DOMAIN, "mp_last_profile: NULL");
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (g_small_prof_ev) { // the last run took the small-N path: its event times, read now
        cudaEvent_t *ev = g_small_prof_ev;
        float kms = 0.f, all = 0.f, setup = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&kms, ev[1], ev[2]));
        all = kms;
        if (g_small_prof_staged) {
            CUDA_TRY(cudaEventElapsedTime(&all, ev[0], ev[3]));
            CUDA_TRY(cudaEventElapsedTime(&setup, ev[0], ev[1]));
        }
        g_prof.product_ms = kms;
        g_prof.spmm_ms = kms;
        g_prof.total_ms = all;
        g_prof.setup_ms = setup;
        g_small_prof_ev = nullptr;
    }
    *out = g_prof;
    return MP_OK;
}

mp_status mp_set_stream(void *stream)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    int dev = 0;
    DevState *st = nullptr;
    TRY(current_device(&dev, &st));
    st->user_stream = (cudaStream_t)stream;
    return MP_OK;
}

mp_status mp_set_options(int sparsity, int64_t device_budget_bytes)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (device_budget_bytes < 0) return fail(MP_ERR_DOMAIN, "mp_set_options: negative budget");
    if (sparsity < -1 || sparsity > 2) return fail(MP_ERR_DOMAIN, "mp_set_options: sparsity %d outside [-1, 2]", sparsity);
    g_opts.sparsity = sparsity;
    g_opts.budget = device_budget_bytes;
    return MP_OK;
}

mp_status mp_set_symmetry(const int32_t *sigma, int64_t N)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!sigma || N <= 0) {
        g_sym.clear();
        ++g_sym_version;
        return MP_OK;
    }
    for (int64_t i = 0; i < N; ++i)
        if (sigma[i] < 0 || sigma[i] >= N || sigma[sigma[i]] != i)
            return fail(MP_ERR_DOMAIN, "mp_set_symmetry: sigma is not an involution of [0, %lld)", (long long)N);
    g_sym.assign(sigma, sigma + N);
    ++g_sym_version;
    return MP_OK;
}

mp_status mp_set_word_symmetry(int on)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    g_word_sym = on != 0;
    g_cache.clear(); // records were computed either way; keep the switch observable
    return MP_OK;
}

mp_status mp_word_reversal(int n, int32_t *sigma_out, int64_t N)
{
    if (n < 2 || n > MP_MAX_N || !sigma_out) return fail(MP_ERR_DOMAIN, "mp_word_reversal: n = %d outside [2, 13]", n);
    const std::vector<int32_t> sg = word_reversal(n);
    if ((int64_t)sg.size() != N)
        return fail(MP_ERR_DOMAIN, "mp_word_reversal: N = %lld, A(D_%d) has %zu words", (long long)N, n, sg.size());
    std::memcpy(sigma_out, sg.data(), sg.size() * 4);
    return MP_OK;
}

mp_status mp_set_transfer_hint(int n)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (n != 0 && (n < 2 || n > MP_MAX_N))
        return fail(MP_ERR_DOMAIN, "mp_set_transfer_hint: n = %d outside {0} u [2, %d]", n, MP_MAX_N);
    g_transfer_n = n;
    return MP_OK;
}

mp_status mp_set_row_reuse(int on)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    g_row_reuse = on != 0;
    g_cache.clear(); // records of the words source were computed either way
    return MP_OK;
}

mp_status mp_set_small_path(int on)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    g_small_off = on == 0;
    return MP_OK;
}

mp_status mp_set_power_observer(mp_power_observer_fn fn, void *ctx)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    g_obs.fn = fn;
    g_obs.ctx = fn ? ctx : nullptr;
    return MP_OK;
}

mp_status mp_set_grouping(int mode)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (mode < -1 || mode > 1) return fail(MP_ERR_DOMAIN, "mp_set_grouping: mode %d outside [-1, 1]", mode);
    g_opts.grouping = mode;
    return MP_OK;
}

mp_status mp_set_spmm_width(int cols)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    const int a = cols < 0 ? -cols : cols;
    if (a != 0 && a != 256 && a != 512 && a != 1024)
        return fail(MP_ERR_DOMAIN, "mp_set_spmm_width: %d is not 0, +-256, +-512 or +-1024", cols);
    g_spmm_width = cols;
    return MP_OK;
}

} // extern "C"
