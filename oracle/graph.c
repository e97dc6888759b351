/*
 * oracle/graph.c -- TEST INFRASTRUCTURE ONLY (see oracle/oracle.c for the rules).
 *
 * gamma_2 of the cylinder P_n x C_m computed on the graph itself, with no transfer matrix,
 * no words and no (min,+) algebra, so that it pins the transfer-matrix oracle (c7):
 *   - oracle_gamma2_bruteforce: every vertex subset, smallest 2-dominating one
 *     ("each vertex not in S has at least two neighbors in it"), n*m <= 26;
 *   - oracle_gamma2_column_dp: the same minimum by dynamic programming over consecutive
 *     column subsets (S_{j-1}, S_j), with (S_0, S_1) fixed to close the cycle, n <= 5.
 * Vertex (i, j): i = row on the path P_n (0..n-1), j = column on the cycle C_m (0..m-1)
 * (with the n/m swap of DESIGN.md G1).  m >= 3 (G17).
 */
#include <stdint.h>
#include <stdlib.h>

static int popc64(uint64_t x) { return __builtin_popcountll(x); }

/* Returns gamma_2, or -1 on bad arguments. */
int oracle_gamma2_bruteforce(int n, int m)
{
    int V = n * m, v, best = V;
    uint64_t nbr[64], S, total;
    if (n < 1 || m < 3 || V > 26) return -1;
    for (v = 0; v < V; v++) {
        int i = v / m, j = v % m;
        uint64_t b = 0;
        if (i > 0) b |= 1ull << ((i - 1) * m + j);
        if (i < n - 1) b |= 1ull << ((i + 1) * m + j);
        b |= 1ull << (i * m + (j + 1) % m);
        b |= 1ull << (i * m + (j + m - 1) % m);
        nbr[v] = b;
    }
    total = 1ull << V;
    for (S = 0; S < total; S++) {
        int size = popc64(S), ok = 1;
        if (size >= best) continue;
        for (v = 0; v < V && ok; v++)
            if (!((S >> v) & 1) && popc64(nbr[v] & S) < 2) ok = 0;
        if (ok) best = size;
    }
    return best;
}

/* Column j (subset cur) is 2-dominated given its neighbouring columns prev and next. */
static int column_ok(int n, unsigned prev, unsigned cur, unsigned next)
{
    int i;
    for (i = 0; i < n; i++) {
        int cnt;
        if ((cur >> i) & 1) continue;
        cnt = ((prev >> i) & 1) + ((next >> i) & 1);
        if (i > 0) cnt += (cur >> (i - 1)) & 1;
        if (i < n - 1) cnt += (cur >> (i + 1)) & 1;
        if (cnt < 2) return 0;
    }
    return 1;
}

/* Row i of the cylinder (the m vertices (i, 0..m-1) of one copy of C_m, as a bit mask cur)
 * is 2-dominated given the rows above (prev) and below (next): every vertex not in S has at
 * least two neighbours in S among its two cycle neighbours and the vertices above/below. */
static int row_ok(int m, unsigned prev, unsigned cur, unsigned next)
{
    int j;
    for (j = 0; j < m; j++) {
        int cnt;
        if ((cur >> j) & 1) continue;
        cnt = ((prev >> j) & 1) + ((next >> j) & 1) + ((cur >> ((j + 1) % m)) & 1) +
              ((cur >> ((j + m - 1) % m)) & 1);
        if (cnt < 2) return 0;
    }
    return 1;
}

/* gamma_2(P_n x C_m) by dynamic programming ALONG THE PATH over consecutive row subsets
 * (S_{i-1}, S_i) of the cycle, with empty virtual rows above row 0 and below row n-1: any
 * path order n, small cycle length 3 <= m <= 8.  Independent of the transfer matrix; it pins
 * the large-n results at small m.  Returns -1 on bad arguments. */
int oracle_gamma2_path_dp(int n, int m)
{
    int C, i, x, y, z, best = 1 << 30;
    int *f, *g;
    unsigned char *ok;
    if (n < 1 || m < 3 || m > 8) return -1;
    C = 1 << m;
    ok = (unsigned char *)malloc((size_t)C * C * C);
    f = (int *)malloc(sizeof(int) * C * C);
    g = (int *)malloc(sizeof(int) * C * C);
    for (x = 0; x < C; x++)
        for (y = 0; y < C; y++)
            for (z = 0; z < C; z++) ok[((size_t)x * C + y) * C + z] = (unsigned char)row_ok(m, x, y, z);
    /* state after placing rows 0..i: (S_{i-1}, S_i); row i-1 already checked */
    for (x = 0; x < C * C; x++) f[x] = 1 << 30;
    for (y = 0; y < C; y++) f[0 * C + y] = __builtin_popcount(y); /* S_{-1} = empty */
    for (i = 1; i < n; i++) {
        for (x = 0; x < C * C; x++) g[x] = 1 << 30;
        for (x = 0; x < C; x++)
            for (y = 0; y < C; y++) {
                int fv = f[x * C + y];
                if (fv >= (1 << 30)) continue;
                for (z = 0; z < C; z++)
                    if (ok[((size_t)x * C + y) * C + z]) {
                        int nv = fv + __builtin_popcount(z);
                        if (nv < g[y * C + z]) g[y * C + z] = nv;
                    }
            }
        { int *t = f; f = g; g = t; }
    }
    for (x = 0; x < C; x++)
        for (y = 0; y < C; y++) {
            int fv = f[x * C + y];
            if (fv < best && ok[((size_t)x * C + y) * C + 0]) best = fv; /* S_n = empty */
        }
    free(ok);
    free(f);
    free(g);
    return best;
}

/* Returns gamma_2, or -1 on bad arguments. */
int oracle_gamma2_column_dp(int n, int m)
{
    int C, a, b, x, y, z, j, best = 1 << 30;
    int *f, *g;
    unsigned char *ok;
    if (n < 1 || n > 5 || m < 3) return -1;
    C = 1 << n;
    ok = (unsigned char *)malloc((size_t)C * C * C);
    f = (int *)malloc(sizeof(int) * C * C);
    g = (int *)malloc(sizeof(int) * C * C);
    for (x = 0; x < C; x++)
        for (y = 0; y < C; y++)
            for (z = 0; z < C; z++) ok[(x * C + y) * C + z] = (unsigned char)column_ok(n, x, y, z);
    for (a = 0; a < C; a++)
        for (b = 0; b < C; b++) {
            /* state after placing S_0 = a, S_1 = b: (S_0, S_1) */
            for (x = 0; x < C * C; x++) f[x] = 1 << 30;
            f[a * C + b] = __builtin_popcount(a) + __builtin_popcount(b);
            for (j = 2; j < m; j++) { /* choose S_j = z, check column j-1 */
                for (x = 0; x < C * C; x++) g[x] = 1 << 30;
                for (x = 0; x < C; x++)
                    for (y = 0; y < C; y++) {
                        int fv = f[x * C + y];
                        if (fv >= (1 << 30)) continue;
                        for (z = 0; z < C; z++)
                            if (ok[(x * C + y) * C + z]) {
                                int nv = fv + __builtin_popcount(z);
                                if (nv < g[y * C + z]) g[y * C + z] = nv;
                            }
                    }
                { int *t = f; f = g; g = t; }
            }
            /* close the cycle: column m-1 sees (S_{m-2}, S_{m-1}, S_0), column 0 sees
             * (S_{m-1}, S_0, S_1) */
            for (x = 0; x < C; x++)
                for (y = 0; y < C; y++) {
                    int fv = f[x * C + y];
                    if (fv >= best) continue;
                    if (ok[(x * C + y) * C + a] && ok[(y * C + a) * C + b]) best = fv;
                }
        }
    free(ok);
    free(f);
    free(g);
    return best;
}
