/*
 * oracle/oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU oracle for the hot path of arXiv 2409.17688
 * ("HPC acceleration of large (min,+) matrix products to compute domination-type
 * parameters in graphs").  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product library
 * (paper_2409_17688_b200/) shares no code, header, table or constant generator with it
 * and never loads it.
 *
 * Citations: "P:L" = reference PAPER.md line L; "S:L" = reference SPEC.md line L;
 * "G<k>" = a reading listed in DESIGN.md section "Readings of the paper".
 *
 * Every function follows the plain definition (or the paper's algorithm in its own
 * order).  The only liberties are the ones DESIGN.md lists:
 *   - the product keeps the definition C_ij = min_k s(A_ik + B_kj) but may visit the
 *     (i,k,j) index space in i-k-j order and skip k with A_ik = inf (min over a set does
 *     not depend on visiting order, and an inf term never wins); oracle_minplus_ijk is the
 *     literal i-j-k loop and the tests pin the two against each other;
 *   - the outer row loop may run on several OpenMP threads (rows are independent; this is
 *     the paper's own OpenMP strategy).
 *
 * Parity status of each function is in its header comment and in DESIGN.md.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_INF 0xFFFFu        /* +inf at the boundary (G6)                 */
#define OR_FINITE_MAX 0x7FFEu /* largest finite value; a finite sum above it is +inf (G6) */

/* ------------------------------------------------------------------------------------ */
/* c1 words.  P:136-139: "words ... containing neither the sequences 020, 111, 211, 112,
 * 212 in any position, nor the sequences 11, 12 at the beginning ... nor the sequences
 * 11, 21 at the end".  P:228: "we first obtain all the m-element variations of 3-elements
 * 0,1,2, with repetition allowed. Then, we select those of them not containing the
 * forbidden sequences".  Order (G5): lexicographic 0<1<2, first letter most significant.
 * Pinned by Table 1, SPEC's m=2 list.                               */
/* ------------------------------------------------------------------------------------ */

int oracle_is_correct_word(const uint8_t *w, int n)
{
    int i;
    for (i = 0; i < n; i++)
        if (w[i] > 2) return -1;
    for (i = 0; i + 2 < n; i++) {
        int a = w[i], b = w[i + 1], c = w[i + 2];
        if (a == 0 && b == 2 && c == 0) return 0; /* 020 */
        if (a == 1 && b == 1 && c == 1) return 0; /* 111 */
        if (a == 2 && b == 1 && c == 1) return 0; /* 211 */
        if (a == 1 && b == 1 && c == 2) return 0; /* 112 */
        if (a == 2 && b == 1 && c == 2) return 0; /* 212 */
    }
    if (n >= 2) {
        if (w[0] == 1 && w[1] == 1) return 0;         /* 11 at the beginning */
        if (w[0] == 1 && w[1] == 2) return 0;         /* 12 at the beginning */
        if (w[n - 2] == 1 && w[n - 1] == 1) return 0; /* 11 at the end */
        if (w[n - 2] == 2 && w[n - 1] == 1) return 0; /* 21 at the end */
    }
    return 1;
}

/* All 3^n variations in lexicographic order, filtered.  If out != NULL it receives the
 * words, n letters each.  Returns the count |C_n|. */
int64_t oracle_words(int n, uint8_t *out)
{
    int64_t total = 1, v, count = 0;
    int i;
    uint8_t w[32];
    if (n < 1 || n > 20) return -1;
    for (i = 0; i < n; i++) total *= 3;
    for (v = 0; v < total; v++) {
        int64_t r = v;
        for (i = n - 1; i >= 0; i--) { /* letter 0 is the most significant digit */
            w[i] = (uint8_t)(r % 3);
            r /= 3;
        }
        if (oracle_is_correct_word(w, n) == 1) {
            if (out) memcpy(out + count * n, w, (size_t)n);
            count++;
        }
    }
    return count;
}

/* c2 can-follow.  P:141-147, rule by rule:
 *   (1) if q_i = 2 then p_i = 0;
 *   (2) if p_i = 2 then exactly one among p_{i-1}, p_{i+1}, q_i is 0 (only the existing
 *       neighbours at i = 1 and i = m, G3);
 *   (3) if p_i = 1 then at least two among them are 0 (at the ends: both, G2).
 * Pinned by S:72-75 and, downstream, Tables 1/4/5/7.                                    */
int oracle_can_follow(const uint8_t *q, const uint8_t *p, int n)
{
    int i;
    for (i = 0; i < n; i++) {
        if (q[i] == 2 && p[i] != 0) return 0; /* rule (1) */
        if (p[i] == 1 || p[i] == 2) {
            int zeros = 0;
            if (i > 0 && p[i - 1] == 0) zeros++;
            if (i < n - 1 && p[i + 1] == 0) zeros++;
            if (q[i] == 0) zeros++;
            if (p[i] == 2 && zeros != 1) return 0; /* rule (2) */
            if (p[i] == 1 && zeros < 2) return 0;  /* rule (3) */
        }
    }
    return 1;
}

/* Arc label: "l(q,p) = number of zeros of p". */
int oracle_zero_count(const uint8_t *p, int n)
{
    int i, z = 0;
    for (i = 0; i < n; i++) z += (p[i] == 0);
    return z;
}

/* c3 Algorithm 1: A_(i,j) = zeros(p_j) if p_j can follow q_i, else inf.
 * A must hold N*N entries, N = oracle_words(n, NULL). Returns N or -1. */
int64_t oracle_transition_matrix(int n, uint16_t *A)
{
    int64_t N = oracle_words(n, NULL), i;
    uint8_t *w;
    if (N <= 0) return -1;
    w = (uint8_t *)malloc((size_t)(N * n));
    if (!w) return -1;
    oracle_words(n, w);
#pragma omp parallel for schedule(dynamic, 16)
    for (i = 0; i < N; i++) {
        int64_t j;
        for (j = 0; j < N; j++) {
            const uint8_t *q = w + i * n, *p = w + j * n;
            A[i * N + j] = oracle_can_follow(q, p, n) ? (uint16_t)oracle_zero_count(p, n)
                                                      : (uint16_t)OR_INF;
        }
    }
    free(w);
    return N;
}

/* ------------------------------------------------------------------------------------ */
/* c4 product.  P:53: (A x B)_ij = min_k (a_ik + b_kj) over (R u {inf}, min, +).
 * 16-bit storage with the saturation reading G6: s(a,b) = a+b if both finite and
 * a+b <= 0x7FFE, else inf; C_ij = min_k s(A_ik, B_kj), starting from inf.
 * Shapes: A is M x K, B is K x N, C is M x N, all row-major contiguous.               */
/* ------------------------------------------------------------------------------------ */

static inline uint32_t sat_add(uint32_t a, uint32_t b)
{
    uint32_t s;
    if (a == OR_INF || b == OR_INF) return OR_INF;
    s = a + b;
    return s <= OR_FINITE_MAX ? s : OR_INF;
}

/* The literal definition: i-j-k loops. */
void oracle_minplus_ijk(const uint16_t *A, const uint16_t *B, uint16_t *C, int64_t M,
                        int64_t K, int64_t N)
{
    int64_t i;
#pragma omp parallel for schedule(static)
    for (i = 0; i < M; i++) {
        int64_t j, k;
        for (j = 0; j < N; j++) {
            uint32_t best = OR_INF;
            for (k = 0; k < K; k++) {
                uint32_t s = sat_add(A[i * K + k], B[k * N + j]);
                if (s < best) best = s;
            }
            C[i * N + j] = (uint16_t)best;
        }
    }
}

/* Same definition, visiting k before j, skipping the k whose A_ik is inf (such a term is
 * inf and never lowers a min).  Used for the large cases; pinned to oracle_minplus_ijk. */
void oracle_minplus_ikj(const uint16_t *A, const uint16_t *B, uint16_t *C, int64_t M,
                        int64_t K, int64_t N)
{
    int64_t i;
#pragma omp parallel for schedule(dynamic, 4)
    for (i = 0; i < M; i++) {
        int64_t j, k;
        uint32_t *row = (uint32_t *)malloc((size_t)N * sizeof(uint32_t));
        for (j = 0; j < N; j++) row[j] = OR_INF;
        for (k = 0; k < K; k++) {
            uint32_t a = A[i * K + k];
            const uint16_t *b = B + k * N;
            if (a == OR_INF) continue;
            for (j = 0; j < N; j++) {
                uint32_t bb = b[j];
                uint32_t s = (bb == OR_INF) ? OR_INF : a + bb;
                if (s < row[j]) row[j] = s;
            }
        }
        for (j = 0; j < N; j++) C[i * N + j] = (uint16_t)(row[j] <= OR_FINITE_MAX ? row[j] : OR_INF);
        free(row);
    }
}

/* ------------------------------------------------------------------------------------ */
/* c4 fingerprint (SURVEY.md section 8(a) note a4):
 *   s(z)   = splitmix64 finaliser of z + 0x9E3779B97F4A7C15;
 *   h(i,j) = s(2i) * s(2j + 1)  (row weight times column weight);
 *   H(X)   = sum over i, j of h(i,j) * x_ij  (mod 2^64), inf encoded as 0xFFFF.
 * Not a paper quantity: a checksum both sides define independently so whole matrices can
 * be compared without moving them.  Pinned by the splitmix64 test vectors, linearity,
 * additivity and single entries. */
/* ------------------------------------------------------------------------------------ */

uint64_t oracle_splitmix64(uint64_t t)
{
    uint64_t z = t + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t oracle_fingerprint(const uint16_t *X, int64_t R, int64_t Ncols)
{
    uint64_t H = 0;
    int64_t i, j;
    for (i = 0; i < R; i++)
        for (j = 0; j < Ncols; j++)
            H += oracle_splitmix64(2 * (uint64_t)i) * oracle_splitmix64(2 * (uint64_t)j + 1) *
                 (uint64_t)X[i * Ncols + j];
    return H;
}

/* Fingerprint of the column block [c0, c1) of an R x Ncols matrix, with the global column
 * index j (the additive shard contribution used by the multi-rank tests). */
uint64_t oracle_fingerprint_cols(const uint16_t *X, int64_t R, int64_t Ncols, int64_t c0,
                                 int64_t c1)
{
    uint64_t H = 0;
    int64_t i, j;
    for (i = 0; i < R; i++)
        for (j = c0; j < c1; j++)
            H += oracle_splitmix64(2 * (uint64_t)i) * oracle_splitmix64(2 * (uint64_t)j + 1) *
                 (uint64_t)X[i * Ncols + j];
    return H;
}

/* ------------------------------------------------------------------------------------ */
/* c5 / c6 / a4: the power sequence (Algorithm 2: A^i = A x A^{i-1}) until the
 * first repeat up to an additive constant (Lemma 1; the hypothesis
 * A^{n0+a} = b x A^{n0} of Theorem 3).  Every power is stored and each new
 * power A^k is compared with every stored A^j, j = k-1 down to 1 (G9: equal inf pattern
 * and a constant difference on the finite entries; if both are all-inf the constant is 0).
 * The first hit gives mu = j, lambda = k - j, b = c.  diag_min[k] = min_i (A^k)_ii
 * (Algorithm 5).  Pinned by Table 5 and the gamma_2 pins.       */
/* ------------------------------------------------------------------------------------ */

typedef struct {
    int32_t mu, lambda, offset, k_last, dense_from;
    uint16_t diag_min[257];
    uint64_t fingerprint[257];
} oracle_periodic_result;

/* Returns 1 and the constant in *c if Y - X is constant on finite entries with equal inf
 * pattern, else 0. */
int oracle_constant_difference(const uint16_t *Y, const uint16_t *X, int64_t count, int32_t *c)
{
    int64_t t;
    int have = 0;
    int32_t d = 0;
    for (t = 0; t < count; t++) {
        int yi = (Y[t] == OR_INF), xi = (X[t] == OR_INF);
        if (yi != xi) return 0;
        if (yi) continue;
        if (!have) {
            d = (int32_t)Y[t] - (int32_t)X[t];
            have = 1;
        } else if ((int32_t)Y[t] - (int32_t)X[t] != d) {
            return 0;
        }
    }
    *c = have ? d : 0;
    return 1;
}

static uint16_t diag_min_of(const uint16_t *X, int64_t N)
{
    int64_t i;
    uint16_t m = OR_INF;
    for (i = 0; i < N; i++)
        if (X[i * N + i] < m) m = X[i * N + i];
    return m;
}

static int has_inf(const uint16_t *X, int64_t count)
{
    int64_t t;
    for (t = 0; t < count; t++)
        if (X[t] == OR_INF) return 1;
    return 0;
}

/* Returns 0 on success, 4 if no repeat with k <= max_k, 1 on bad arguments, 3 on
 * allocation failure. */
int oracle_power_until_periodic(const uint16_t *A, int64_t N, int max_k, oracle_periodic_result *out)
{
    uint16_t **P;
    int k, j, rc = 4;
    size_t bytes = (size_t)N * (size_t)N * sizeof(uint16_t);
    if (N <= 0 || max_k < 2 || max_k > 256 || !out) return 1;
    memset(out, 0, sizeof(*out));
    P = (uint16_t **)calloc((size_t)max_k + 1, sizeof(uint16_t *));
    if (!P) return 3;
    P[1] = (uint16_t *)malloc(bytes);
    if (!P[1]) { free(P); return 3; }
    memcpy(P[1], A, bytes);
    out->diag_min[1] = diag_min_of(P[1], N);
    out->fingerprint[1] = oracle_fingerprint(P[1], N, N);
    if (!has_inf(P[1], N * N)) out->dense_from = 1;
    for (k = 2; k <= max_k; k++) {
        P[k] = (uint16_t *)malloc(bytes);
        if (!P[k]) { rc = 3; break; }
        oracle_minplus_ikj(A, P[k - 1], P[k], N, N, N); /* A^k = A x A^{k-1} */
        out->diag_min[k] = diag_min_of(P[k], N);
        out->fingerprint[k] = oracle_fingerprint(P[k], N, N);
        if (!out->dense_from && !has_inf(P[k], N * N)) out->dense_from = k;
        for (j = k - 1; j >= 1; j--) {
            int32_t c;
            if (oracle_constant_difference(P[k], P[j], N * N, &c)) {
                out->mu = j;
                out->lambda = k - j;
                out->offset = c;
                out->k_last = k;
                rc = 0;
                break;
            }
        }
        if (rc == 0) break;
    }
    if (rc != 0) out->k_last = (k > max_k) ? max_k : k;
    for (k = 1; k <= max_k; k++) free(P[k]);
    free(P);
    return rc;
}

/* Row r of every power A^1..A^kmax, by repeated (min,+) vector-matrix products
 * e_r^T A^k = (e_r^T A^{k-1}) x A (associativity).  rows_out holds kmax*N entries; row k-1
 * is row r of A^k.  Used to check sampled outputs at sizes where full powers are too big
 * for the oracle (n = 11, 12).  cur_j = min_l s(prev_l + A_lj): the l loop runs inside
 * column chunks (the minimum over l does not depend on the visiting order); an inf term is
 * carried as a sum >= 0xFFFF and mapped to inf by the final clamp, which is s() of G6.   */
void oracle_power_rows(const uint16_t *A, int64_t N, int64_t r, int kmax, uint16_t *rows_out)
{
    int k;
    memcpy(rows_out, A + r * N, (size_t)N * sizeof(uint16_t));
    for (k = 2; k <= kmax; k++) {
        const uint16_t *prev = rows_out + (int64_t)(k - 2) * N;
        uint16_t *cur = rows_out + (int64_t)(k - 1) * N;
        int64_t jc;
#pragma omp parallel for schedule(dynamic, 1)
        for (jc = 0; jc < N; jc += 2048) {
            const int64_t je = (jc + 2048 < N) ? jc + 2048 : N;
            uint32_t acc[2048];
            int64_t j, l;
            for (j = jc; j < je; j++) acc[j - jc] = OR_INF;
            for (l = 0; l < N; l++) {
                const uint32_t a = prev[l];
                const uint16_t *Arow = A + l * N;
                if (a == OR_INF) continue;
                for (j = jc; j < je; j++) {
                    const uint32_t s = a + Arow[j]; /* >= 0xFFFF when A_lj is inf */
                    if (s < acc[j - jc]) acc[j - jc] = s;
                }
            }
            for (j = jc; j < je; j++)
                cur[j] = (uint16_t)(acc[j - jc] <= OR_FINITE_MAX ? acc[j - jc] : OR_INF);
        }
    }
}

/* a6 read-off (Theorem 2; Theorem 3):
 * gamma_2(P_n x C_m) = diag_min[m] if m <= k_last, else diag_min[m - t*lambda] + t*b with
 * t the least integer that brings m - t*lambda into [mu, k_last].  Returns -1 if m < 3
 * (G17). */
int64_t oracle_gamma2_readoff(const oracle_periodic_result *r, int64_t m)
{
    int64_t t;
    if (m < 3) return -1;
    if (m <= r->k_last) return r->diag_min[m];
    t = (m - r->k_last + r->lambda - 1) / r->lambda;
    return (int64_t)r->diag_min[m - t * r->lambda] + t * (int64_t)r->offset;
}

int oracle_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
