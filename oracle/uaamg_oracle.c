/*
 * uaamg_oracle.c -- CPU restatement of the reference UA-AMG setup/solve path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("port") for the B200 build; nothing in paper_1302_2547_b200/
 * links or calls it.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.
 *
 * Every function restates one piece of the reference package
 * (/root/reference/pkg/src/uaamg, "U/" below; "K/" = U/kernels/) and cites
 * the file:line it follows.  Index arrays are int64 and values float64, as in
 * the reference SparseMatrix (U/sparse.py:25-27).  Floating-point sums are
 * sequential in the reference's order and the file is compiled with
 * -ffp-contract=off, so every kernel is bit-identical to the numba backend
 * (K/numba_backend.py) for any OpenMP thread count.  Parallel loops mirror the
 * numba prange loops; loops the reference runs serially stay serial except
 * squared_pattern, which is row-independent and is parallelised here with
 * per-thread stamp arrays (same output).
 *
 * Pinning: tests/test_oracle_golden.py checks this oracle bit-for-bit against
 * fixtures produced by running the reference itself (tests/golden/make_golden.py).
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t i64;
typedef uint64_t u64;
typedef uint8_t u8;

/* ------------------------------------------------------------------ */
/* error reporting                                                      */
/* ------------------------------------------------------------------ */
static char g_err[512];
const char *orc_last_error(void) { return g_err; }
static void set_err(const char *msg) { snprintf(g_err, sizeof g_err, "%s", msg); }

void orc_set_num_threads(int n) { omp_set_num_threads(n < 1 ? 1 : n); }
int orc_get_num_threads(void) { return omp_get_max_threads(); }
void orc_free(void *p) { free(p); }

/* ------------------------------------------------------------------ */
/* counter hash  (K/numba_backend.py:14-18 constants, :25-35 mix/hash)  */
/* ------------------------------------------------------------------ */
#define MIX1 0xBF58476D1CE4E5B9ULL
#define MIX2 0x94D049BB133111EBULL
#define PHI 0x9E3779B97F4A7C15ULL
#define PASS_SALT 0xA0761D6478BD642FULL

static inline u64 mix64(u64 z) {
    z = (z ^ (z >> 30)) * MIX1;
    z = (z ^ (z >> 27)) * MIX2;
    return z ^ (z >> 31);
}
static inline u64 pass_base(u64 seed, i64 pass_idx) {
    /* K/numba_backend.py:40 and :103 */
    return mix64(seed ^ (PASS_SALT * (u64)(pass_idx + 1)));
}
static inline double hash_unit(u64 base, i64 i) {
    u64 z = mix64(mix64(base + (u64)i * PHI));
    return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

/* K/numba_backend.py:38-44 */
void orc_hash_u01(u64 seed, i64 pass_idx, const i64 *idx, i64 m, double *out) {
    u64 base = pass_base(seed, pass_idx);
#pragma omp parallel for schedule(static)
    for (i64 k = 0; k < m; k++) out[k] = hash_unit(base, idx[k]);
}

/* ------------------------------------------------------------------ */
/* CSR kernels                                                          */
/* ------------------------------------------------------------------ */
/* K/numba_backend.py:47-56 -- per-row sequential sum, no FMA */
void orc_spmv(i64 n, const i64 *ip, const i64 *ix, const double *a, const double *x, double *y) {
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < n; i++) {
        double acc = 0.0;
        for (i64 k = ip[i]; k < ip[i + 1]; k++) acc += a[k] * x[ix[k]];
        y[i] = acc;
    }
}

/* K/numba_backend.py:59-68 */
void orc_diag_of(i64 n, const i64 *ip, const i64 *ix, const double *a, double *out) {
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < n; i++) {
        double d = 0.0;
        for (i64 k = ip[i]; k < ip[i + 1]; k++)
            if (ix[k] == i) { d = a[k]; break; }
        out[i] = d;
    }
}

/* K/numba_backend.py:71-84 -- M_ii = sum_{j!=i}|a_ij| + a_ii (that add order) */
void orc_l1_diag(i64 n, const i64 *ip, const i64 *ix, const double *a, double *out) {
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < n; i++) {
        double acc = 0.0, dii = 0.0;
        for (i64 k = ip[i]; k < ip[i + 1]; k++) {
            if (ix[k] == i) dii = a[k];
            else acc += fabs(a[k]);
        }
        out[i] = acc + dii;
    }
}

/* K/numba_backend.py:87-97 */
void orc_degrees(i64 n, const i64 *ip, const i64 *ix, i64 *out) {
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < n; i++) {
        i64 d = 0;
        for (i64 k = ip[i]; k < ip[i + 1]; k++) d += (ix[k] != i);
        out[i] = d;
    }
}

/* K/numba_backend.py:100-111 ; U/aggregation.py:130-133
 * v_i = d_i + ((i mod 12) + u_i) / 12, evaluated in exactly that order. */
void orc_scores(i64 n, const i64 *ip, const i64 *ix, u64 seed, i64 pass_idx, double *out) {
    u64 base = pass_base(seed, pass_idx);
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < n; i++) {
        i64 d = 0;
        for (i64 k = ip[i]; k < ip[i + 1]; k++) d += (ix[k] != i);
        out[i] = (double)d + (((double)(i % 12) + hash_unit(base, i)) / 12.0);
    }
}

static int cmp_i64(const void *x, const void *y) {
    i64 a = *(const i64 *)x, b = *(const i64 *)y;
    return (a > b) - (a < b);
}
static void sort_i64(i64 *v, i64 m) {
    if (m < 24) {
        for (i64 s = 1; s < m; s++) {
            i64 t = v[s], p = s - 1;
            while (p >= 0 && v[p] > t) { v[p + 1] = v[p]; p--; }
            v[p + 1] = t;
        }
    } else {
        qsort(v, (size_t)m, sizeof(i64), cmp_i64);
    }
}

/* K/numba_backend.py:114-142 (U/sparse.py:121-129): symbolic A*A pattern,
 * sorted rows.  Row-parallel with per-thread stamps (output identical). */
i64 orc_squared_pattern(i64 n, const i64 *ip, const i64 *ix, i64 **out_ptr, i64 **out_idx) {
    i64 *ptr = (i64 *)calloc((size_t)n + 1, sizeof(i64));
    int nt = omp_get_max_threads();
    /* per-thread stamps hold row indices (< 2^31 for every config): int32
     * halves the n * threads footprint (17 GB at 512^3 with 16 threads) */
    int32_t *stamps = (int32_t *)malloc(sizeof(int32_t) * (size_t)n * (size_t)nt);
    for (i64 s = 0; s < n * (i64)nt; s++) stamps[s] = -1;
#pragma omp parallel
    {
        int32_t *stamp = stamps + (i64)omp_get_thread_num() * n;
#pragma omp for schedule(dynamic, 1024)
        for (i64 i = 0; i < n; i++) {
            i64 cnt = 0;
            for (i64 k = ip[i]; k < ip[i + 1]; k++) {
                i64 kk = ix[k];
                for (i64 k2 = ip[kk]; k2 < ip[kk + 1]; k2++) {
                    i64 j = ix[k2];
                    if (stamp[j] != (int32_t)i) { stamp[j] = (int32_t)i; cnt++; }
                }
            }
            ptr[i + 1] = cnt;
        }
    }
    for (i64 i = 0; i < n; i++) ptr[i + 1] += ptr[i];
    i64 *idx = (i64 *)malloc(sizeof(i64) * (size_t)(ptr[n] > 0 ? ptr[n] : 1));
    for (i64 s = 0; s < n * (i64)nt; s++) stamps[s] = -1;
#pragma omp parallel
    {
        int32_t *stamp = stamps + (i64)omp_get_thread_num() * n;
#pragma omp for schedule(dynamic, 1024)
        for (i64 i = 0; i < n; i++) {
            i64 pos = ptr[i];
            for (i64 k = ip[i]; k < ip[i + 1]; k++) {
                i64 kk = ix[k];
                for (i64 k2 = ip[kk]; k2 < ip[kk + 1]; k2++) {
                    i64 j = ix[k2];
                    if (stamp[j] != (int32_t)i) { stamp[j] = (int32_t)i; idx[pos++] = j; }
                }
            }
            sort_i64(idx + ptr[i], pos - ptr[i]);
        }
    }
    free(stamps);
    *out_ptr = ptr;
    *out_idx = idx;
    return ptr[n];
}

/* K/numba_backend.py:145-172 (U/hierarchy.py:22-28): coarse entry (I,J) is
 * the sequential sum, in original CSR order, of the fine entries keyed
 * v2a[row]*nc + v2a[col]; the stable (mergesort) order is reproduced by a
 * stable LSD radix sort.  Exact zero sums are dropped. */
i64 orc_galerkin(i64 n, const i64 *ip, const i64 *ix, const double *a, const i64 *v2a, i64 nc,
                 i64 **out_ptr, i64 **out_idx, double **out_val) {
    i64 nnz = ip[n];
    i64 *key = (i64 *)malloc(sizeof(i64) * (size_t)(nnz ? nnz : 1));
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < n; i++) {
        i64 base = v2a[i] * nc;
        for (i64 k = ip[i]; k < ip[i + 1]; k++) key[k] = base + v2a[ix[k]];
    }
    i64 *ord = (i64 *)malloc(sizeof(i64) * (size_t)(nnz ? nnz : 1));
    i64 *tmp = (i64 *)malloc(sizeof(i64) * (size_t)(nnz ? nnz : 1));
    for (i64 k = 0; k < nnz; k++) ord[k] = k;
    u64 maxkey = (u64)(nc > 0 ? nc * nc : 1);
    i64 *cnt = (i64 *)malloc(sizeof(i64) * 65536);
    for (int shift = 0; shift < 64 && (maxkey >> shift) > 0; shift += 16) {
        memset(cnt, 0, sizeof(i64) * 65536);
        for (i64 k = 0; k < nnz; k++) cnt[((u64)key[ord[k]] >> shift) & 0xFFFF]++;
        i64 run = 0;
        for (int d = 0; d < 65536; d++) { i64 c = cnt[d]; cnt[d] = run; run += c; }
        for (i64 k = 0; k < nnz; k++) tmp[cnt[((u64)key[ord[k]] >> shift) & 0xFFFF]++] = ord[k];
        i64 *sw = ord; ord = tmp; tmp = sw;
    }
    free(cnt);
    i64 *ptr = (i64 *)calloc((size_t)nc + 1, sizeof(i64));
    i64 *idx = (i64 *)malloc(sizeof(i64) * (size_t)(nnz ? nnz : 1));
    double *val = (double *)malloc(sizeof(double) * (size_t)(nnz ? nnz : 1));
    i64 m = 0, k = 0;
    while (k < nnz) {
        i64 cur = key[ord[k]];
        double acc = 0.0;
        while (k < nnz && key[ord[k]] == cur) { acc += a[ord[k]]; k++; }
        if (acc != 0.0) {
            idx[m] = cur % nc;
            val[m] = acc;
            ptr[cur / nc + 1]++;
            m++;
        }
    }
    for (i64 i = 0; i < nc; i++) ptr[i + 1] += ptr[i];
    free(key); free(ord); free(tmp);
    *out_ptr = ptr; *out_idx = idx; *out_val = val;
    return m;
}

/* K/numba_backend.py:175-193 (U/aggregation.py:136-141) */
void orc_select_centers(i64 n, const i64 *p2, const i64 *x2, const double *s, const u8 *processed, u8 *out) {
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < n; i++) {
        if (processed[i]) { out[i] = 0; continue; }
        int ok = 1;
        double si = s[i];
        for (i64 k = p2[i]; k < p2[i + 1]; k++) {
            i64 j = x2[k];
            if (j == i || processed[j]) continue;
            double sj = s[j];
            if (!(si > sj || (si == sj && i < j))) { ok = 0; break; }
        }
        out[i] = (u8)ok;
    }
}

/* K/numba_backend.py:196-220 */
void orc_claim_owners(i64 n, const i64 *p2, const i64 *x2, const double *s, const u8 *processed,
                      const u8 *is_center, i64 *owner) {
#pragma omp parallel for schedule(static)
    for (i64 j = 0; j < n; j++) {
        if (is_center[j]) { owner[j] = j; continue; }
        owner[j] = -1;
        if (processed[j]) continue;
        i64 best = -1;
        double best_s = 0.0, sj = s[j];
        for (i64 k = p2[j]; k < p2[j + 1]; k++) {
            i64 i = x2[k];
            if (!is_center[i]) continue;
            double si = s[i];
            if (si < sj) continue;
            if (best == -1 || si > best_s || (si == best_s && i < best)) { best = i; best_s = si; }
        }
        owner[j] = best;
    }
}

/* The same two functions without forming A^2: the maximum over the
 * distance-2 neighbourhood as two maximum hops over A (key = (s, -index)).
 * select: i is a center iff unprocessed and the best unprocessed key within
 * distance 2 is i's own (or there is none better); claim: the best center
 * within distance 2, kept iff its score >= s_j (the best key has the best
 * score, so this equals the pattern loops' filter-then-max).  Identical
 * results (tests/test_oracle_golden.py checks both modes on every fixture);
 * used when A^2 would not fit in memory -- C5 (512^3) has coarse levels with
 * hub rows whose A^2 rows span the whole level. */
static inline int key_gt(double sa, i64 ia, double sb, i64 ib) { return sa > sb || (sa == sb && ia < ib); }
static void hop_max(i64 n, const i64 *ip, const i64 *ix, const double *s, const u8 *ok, double *ms, i64 *mi) {
#pragma omp parallel for schedule(static)
    for (i64 k = 0; k < n; k++) {
        double bs = 0.0;
        i64 bi = -1;
        for (i64 e = ip[k]; e < ip[k + 1]; e++) {
            i64 j = ix[e];
            if (!ok[j]) continue;
            if (bi < 0 || key_gt(s[j], j, bs, bi)) { bs = s[j]; bi = j; }
        }
        ms[k] = bs;
        mi[k] = bi;
    }
}
static void hop2_best(const i64 *ip, const i64 *ix, const double *ms, const i64 *mi, i64 i, double *bs, i64 *bi) {
    *bs = 0.0;
    *bi = -1;
    for (i64 e = ip[i]; e < ip[i + 1]; e++) {
        i64 k = ix[e], c = mi[k];
        if (c < 0) continue;
        if (*bi < 0 || key_gt(ms[k], c, *bs, *bi)) { *bs = ms[k]; *bi = c; }
    }
}
void orc_select_centers_2hop(i64 n, const i64 *ip, const i64 *ix, const double *s, const u8 *processed, u8 *out) {
    u8 *ok = (u8 *)malloc((size_t)n);
    double *ms = (double *)malloc(sizeof(double) * (size_t)n);
    i64 *mi = (i64 *)malloc(sizeof(i64) * (size_t)n);
    for (i64 j = 0; j < n; j++) ok[j] = !processed[j];
    hop_max(n, ip, ix, s, ok, ms, mi);
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < n; i++) {
        if (processed[i]) { out[i] = 0; continue; }
        double bs;
        i64 bi;
        hop2_best(ip, ix, ms, mi, i, &bs, &bi);
        out[i] = (u8)(bi < 0 || bi == i || key_gt(s[i], i, bs, bi));
    }
    free(ok); free(ms); free(mi);
}
void orc_claim_owners_2hop(i64 n, const i64 *ip, const i64 *ix, const double *s, const u8 *processed,
                           const u8 *is_center, i64 *owner) {
    double *ms = (double *)malloc(sizeof(double) * (size_t)n);
    i64 *mi = (i64 *)malloc(sizeof(i64) * (size_t)n);
    hop_max(n, ip, ix, s, is_center, ms, mi);
#pragma omp parallel for schedule(static)
    for (i64 j = 0; j < n; j++) {
        if (is_center[j]) { owner[j] = j; continue; }
        owner[j] = -1;
        if (processed[j]) continue;
        double bs;
        i64 bi;
        hop2_best(ip, ix, ms, mi, j, &bs, &bi);
        owner[j] = (bi >= 0 && !(bs < s[j])) ? bi : -1;
    }
    free(ms); free(mi);
}

/* 0: A^2 pattern unless it would exceed kA2MaxEntries, 1: always A^2, 2: always two hops */
static int g_select_mode = 0;
void orc_set_select_mode(int m) { g_select_mode = m; }
static const i64 kA2MaxEntries = (i64)1 << 29; /* 4 GB of int64 indices */

/* lower_bound in a sorted i64 range */
static inline i64 lower_bound(const i64 *v, i64 lo, i64 hi, i64 key) {
    while (lo < hi) {
        i64 mid = lo + (hi - lo) / 2;
        if (v[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

/* stable ascending argsort of doubles (mergesort semantics) */
static void stable_argsort(const double *w, i64 m, i64 *ord, i64 *tmp) {
    for (i64 t = 0; t < m; t++) ord[t] = t;
    for (i64 width = 1; width < m; width *= 2) {
        for (i64 lo = 0; lo < m; lo += 2 * width) {
            i64 mid = lo + width < m ? lo + width : m;
            i64 hi = lo + 2 * width < m ? lo + 2 * width : m;
            i64 p = lo, q = mid, o = lo;
            while (p < mid && q < hi) tmp[o++] = (w[ord[q]] < w[ord[p]]) ? ord[q++] : ord[p++];
            while (p < mid) tmp[o++] = ord[p++];
            while (q < hi) tmp[o++] = ord[q++];
        }
        memcpy(ord, tmp, sizeof(i64) * (size_t)m);
    }
}

/* K/numba_backend.py:223-273: per center, candidates ordered by descending
 * |A_cj| (stable), repeated sweeps admitting a candidate when its row touches
 * the center or an admitted candidate, until the cap or no progress. */
void orc_admit_members(const i64 *ip, const i64 *ix, const double *a, i64 nctr, const i64 *centers,
                       const i64 *bptr, const i64 *bjs, i64 cap, u8 *processed, i64 *v2a, i64 agg_base) {
#pragma omp parallel for schedule(dynamic, 64)
    for (i64 b = 0; b < nctr; b++) {
        i64 c = centers[b];
        i64 agg = agg_base + b;
        v2a[c] = agg;
        processed[c] = 1;
        i64 lo = bptr[b], hi = bptr[b + 1], m = hi - lo;
        if (m == 0) continue;
        const i64 *js = bjs + lo;
        double *w = (double *)malloc(sizeof(double) * (size_t)m);
        i64 *ord = (i64 *)malloc(sizeof(i64) * (size_t)m);
        i64 *tmp = (i64 *)malloc(sizeof(i64) * (size_t)m);
        u8 *adm = (u8 *)calloc((size_t)m, 1);
        i64 s = ip[c], e = ip[c + 1];
        for (i64 t = 0; t < m; t++) {
            i64 pos = lower_bound(ix, s, e, js[t]);
            double wv = (pos < e && ix[pos] == js[t]) ? fabs(a[pos]) : 0.0;
            w[t] = -wv;
        }
        stable_argsort(w, m, ord, tmp);
        i64 count = 1;
        int progress = 1;
        while (progress && count < cap) {
            progress = 0;
            for (i64 t = 0; t < m; t++) {
                if (count >= cap) break;
                i64 id = ord[t];
                if (adm[id]) continue;
                i64 j = js[id];
                int conn = 0;
                for (i64 k = ip[j]; k < ip[j + 1]; k++) {
                    i64 nb = ix[k];
                    if (nb == c) { conn = 1; break; }
                    i64 pos = lower_bound(js, 0, m, nb);
                    if (pos < m && js[pos] == nb && adm[pos]) { conn = 1; break; }
                }
                if (conn) {
                    adm[id] = 1;
                    v2a[j] = agg;
                    processed[j] = 1;
                    count++;
                    progress = 1;
                }
            }
        }
        free(w); free(ord); free(tmp); free(adm);
    }
}

/* K/numba_backend.py:276-285 -- ascending member order */
void orc_restrict(i64 nc, const i64 *aptr, const i64 *mem, const double *r, double *out) {
#pragma omp parallel for schedule(static)
    for (i64 I = 0; I < nc; I++) {
        double acc = 0.0;
        for (i64 k = aptr[I]; k < aptr[I + 1]; k++) acc += r[mem[k]];
        out[I] = acc;
    }
}

/* K/numba_backend.py:288-294 */
void orc_prolongate_add(i64 n, const i64 *v2a, const double *ec, const double *x, double *out) {
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < n; i++) out[i] = x[i] + ec[v2a[i]];
}

/* K/numba_backend.py:297-310 -- x is updated in place (caller copies) */
void orc_smooth_sweeps(i64 n, const i64 *ip, const i64 *ix, const double *a, const double *inv_m,
                       double *x, const double *b, i64 sweeps, double *r) {
    for (i64 s = 0; s < sweeps; s++) {
#pragma omp parallel for schedule(static)
        for (i64 i = 0; i < n; i++) {
            double acc = 0.0;
            for (i64 k = ip[i]; k < ip[i + 1]; k++) acc += a[k] * x[ix[k]];
            r[i] = b[i] - acc;
        }
#pragma omp parallel for schedule(static)
        for (i64 i = 0; i < n; i++) x[i] = x[i] + inv_m[i] * r[i];
    }
}

/* ------------------------------------------------------------------ */
/* aggregation driver  (U/aggregation.py:144-203)                       */
/* ------------------------------------------------------------------ */
/* Returns n_coarse (>0) and fills v2a[n] (renumbered) and seeds[n] (first
 * n_coarse entries, strictly increasing); -1 on error.  pass_centers, when
 * non-NULL, receives per vertex the pass index in which it was selected as a
 * center (-1 otherwise) -- a diagnostic for per-pass parity tests. */
i64 orc_aggregate(i64 n, const i64 *ip, const i64 *ix, const double *a, u64 seed, i64 max_passes,
                  i64 cap, i64 *v2a_out, i64 *seeds_out, i64 *pass_centers) {
    if (n <= 0) { set_err("cannot aggregate an empty matrix"); return -1; }
    if (cap <= 0) cap = (i64)1 << 62; /* U/aggregation.py:18,165 */
    /* bound on nnz(A^2): sum over rows of the lengths of the rows they reference */
    i64 bound = 0;
#pragma omp parallel for reduction(+ : bound) schedule(static)
    for (i64 i = 0; i < n; i++)
        for (i64 k = ip[i]; k < ip[i + 1]; k++) bound += ip[ix[k] + 1] - ip[ix[k]];
    const int two_hop = g_select_mode == 2 || (g_select_mode == 0 && bound > kA2MaxEntries);
    i64 *p2 = NULL, *x2 = NULL;
    if (!two_hop) orc_squared_pattern(n, ip, ix, &p2, &x2);
    u8 *processed = (u8 *)calloc((size_t)n, 1);
    u8 *is_center = (u8 *)calloc((size_t)n, 1);
    i64 *v2a = (i64 *)malloc(sizeof(i64) * (size_t)n);
    i64 *owner = (i64 *)malloc(sizeof(i64) * (size_t)n);
    i64 *rank = (i64 *)malloc(sizeof(i64) * (size_t)n);
    i64 *centers = (i64 *)malloc(sizeof(i64) * (size_t)n);
    i64 *all = (i64 *)malloc(sizeof(i64) * (size_t)n);
    i64 *bptr = (i64 *)malloc(sizeof(i64) * ((size_t)n + 1));
    i64 *bjs = (i64 *)malloc(sizeof(i64) * (size_t)n);
    double *s = (double *)malloc(sizeof(double) * (size_t)n);
    i64 nall = 0;
    for (i64 i = 0; i < n; i++) { v2a[i] = -1; if (pass_centers) pass_centers[i] = -1; }
    for (i64 pass = 0; pass < max_passes; pass++) {
        i64 left = 0;
        for (i64 i = 0; i < n; i++) left += !processed[i];
        if (left == 0) break;
        orc_scores(n, ip, ix, seed, pass, s);
        if (two_hop) orc_select_centers_2hop(n, ip, ix, s, processed, is_center);
        else orc_select_centers(n, p2, x2, s, processed, is_center);
        i64 nctr = 0;
        for (i64 i = 0; i < n; i++)
            if (is_center[i]) { rank[i] = nctr; centers[nctr++] = i; }
        if (nctr == 0) break;
        if (pass_centers)
            for (i64 b = 0; b < nctr; b++) pass_centers[centers[b]] = pass;
        if (two_hop) orc_claim_owners_2hop(n, ip, ix, s, processed, is_center, owner);
        else orc_claim_owners(n, p2, x2, s, processed, is_center, owner);
        /* buckets: claimed non-centers grouped by owner rank, ascending j
         * (U/aggregation.py:157-164) */
        memset(bptr, 0, sizeof(i64) * ((size_t)nctr + 1));
        for (i64 j = 0; j < n; j++)
            if (owner[j] >= 0 && !is_center[j]) bptr[rank[owner[j]] + 1]++;
        for (i64 b = 0; b < nctr; b++) bptr[b + 1] += bptr[b];
        for (i64 j = 0; j < n; j++)
            if (owner[j] >= 0 && !is_center[j]) bjs[bptr[rank[owner[j]]]++] = j;
        for (i64 b = nctr; b > 0; b--) bptr[b] = bptr[b - 1];
        bptr[0] = 0;
        orc_admit_members(ip, ix, a, nctr, centers, bptr, bjs, cap, processed, v2a, nall);
        for (i64 b = 0; b < nctr; b++) { all[nall++] = centers[b]; is_center[centers[b]] = 0; }
    }
    /* leftovers become singletons (U/aggregation.py:195-198) */
    for (i64 v = 0; v < n; v++)
        if (!processed[v]) { v2a[v] = nall; all[nall++] = v; }
    /* renumber by ascending seed (U/aggregation.py:199-203) */
    for (i64 k = 0; k < nall; k++) rank[k] = k;
    memcpy(seeds_out, all, sizeof(i64) * (size_t)nall);
    sort_i64(seeds_out, nall);
    /* new_id[k] for old agg k: position of all[k] in the sorted seeds */
    for (i64 k = 0; k < nall; k++) rank[k] = lower_bound(seeds_out, 0, nall, all[k]);
    for (i64 v = 0; v < n; v++) v2a_out[v] = rank[v2a[v]];
    free(p2); free(x2); free(processed); free(is_center); free(v2a); free(owner); free(rank);
    free(centers); free(all); free(bptr); free(bjs); free(s);
    return nall;
}

/* ------------------------------------------------------------------ */
/* hierarchy  (U/hierarchy.py)                                          */
/* ------------------------------------------------------------------ */
typedef struct {
    i64 n, nnz;
    i64 *ip, *ix;
    double *a;
    i64 nc;      /* aggregation to the next level; 0 on the coarsest */
    i64 *v2a, *seeds;
    i64 *mptr, *mem; /* members_csr (U/aggregation.py:70-77) */
} orc_level;

typedef struct {
    int nlev;
    orc_level lev[64];
    int singular;       /* hierarchy flag (U/hierarchy.py:131,152) */
    int coarse_mode;    /* 0 empty, 1 Cholesky, 2 eigen pinv (U/hierarchy.py:31-65) */
    i64 cn;
    double *cfac;       /* Cholesky factor (upper, row-major) or pinv matrix */
} orc_hier;

static void build_members(orc_level *L) {
    /* stable argsort of v2a == counting sort in ascending vertex order */
    L->mptr = (i64 *)calloc((size_t)L->nc + 1, sizeof(i64));
    L->mem = (i64 *)malloc(sizeof(i64) * (size_t)(L->n ? L->n : 1));
    for (i64 i = 0; i < L->n; i++) L->mptr[L->v2a[i] + 1]++;
    for (i64 I = 0; I < L->nc; I++) L->mptr[I + 1] += L->mptr[I];
    i64 *cur = (i64 *)malloc(sizeof(i64) * (size_t)(L->nc ? L->nc : 1));
    memcpy(cur, L->mptr, sizeof(i64) * (size_t)L->nc);
    for (i64 i = 0; i < L->n; i++) L->mem[cur[L->v2a[i]]++] = i;
    free(cur);
}

/* U/hierarchy.py:112-117 */
static int detect_singular(i64 n, const i64 *ip, const i64 *ix, const double *a) {
    i64 nnz = ip[n];
    if (nnz == 0) return 1;
    double scale = 0.0;
    for (i64 k = 0; k < nnz; k++) if (fabs(a[k]) > scale) scale = fabs(a[k]);
    double *one = (double *)malloc(sizeof(double) * (size_t)(n ? n : 1)), *y = (double *)malloc(sizeof(double) * (size_t)n);
    for (i64 i = 0; i < n; i++) one[i] = 1.0;
    orc_spmv(n, ip, ix, a, one, y);
    double mx = 0.0;
    for (i64 i = 0; i < n; i++) if (fabs(y[i]) > mx) mx = fabs(y[i]);
    free(one); free(y);
    return mx <= 1e-10 * scale;
}

/* cyclic Jacobi eigen-decomposition of a symmetric matrix (row-major),
 * eigenvectors in columns of V; stands in for numpy.linalg.eigh */
static void jacobi_eigh(i64 n, double *A, double *V, double *w) {
    for (i64 i = 0; i < n; i++) for (i64 j = 0; j < n; j++) V[i * n + j] = (i == j);
    for (int sweep = 0; sweep < 100; sweep++) {
        double off = 0.0, tot = 0.0;
        for (i64 i = 0; i < n; i++) for (i64 j = 0; j < n; j++) {
            double v = A[i * n + j] * A[i * n + j];
            tot += v;
            if (i != j) off += v;
        }
        if (off <= 1e-30 * (tot > 0 ? tot : 1.0)) break;
        for (i64 p = 0; p < n; p++) for (i64 q = p + 1; q < n; q++) {
            double apq = A[p * n + q];
            if (fabs(apq) < 1e-300) continue;
            double app = A[p * n + p], aqq = A[q * n + q];
            double theta = (aqq - app) / (2.0 * apq);
            double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
            double c = 1.0 / sqrt(t * t + 1.0), sn = t * c;
            for (i64 k = 0; k < n; k++) {
                double akp = A[k * n + p], akq = A[k * n + q];
                A[k * n + p] = c * akp - sn * akq;
                A[k * n + q] = sn * akp + c * akq;
            }
            for (i64 k = 0; k < n; k++) {
                double apk = A[p * n + k], aqk = A[q * n + k];
                A[p * n + k] = c * apk - sn * aqk;
                A[q * n + k] = sn * apk + c * aqk;
            }
            for (i64 k = 0; k < n; k++) {
                double vkp = V[k * n + p], vkq = V[k * n + q];
                V[k * n + p] = c * vkp - sn * vkq;
                V[k * n + q] = sn * vkp + c * vkq;
            }
        }
    }
    for (i64 i = 0; i < n; i++) w[i] = A[i * n + i];
}

/* U/hierarchy.py:31-55: Cholesky if SPD else eigen pseudo-inverse with cut
 * 1e-12*max(lambda_max,0) */
static void coarse_factor(orc_hier *h) {
    orc_level *L = &h->lev[h->nlev - 1];
    i64 n = L->n;
    h->cn = n;
    h->coarse_mode = 0;
    if (n == 0) return;
    double *D = (double *)calloc((size_t)(n * n), sizeof(double));
    for (i64 i = 0; i < n; i++)
        for (i64 k = L->ip[i]; k < L->ip[i + 1]; k++) D[i * n + L->ix[k]] = L->a[k];
    if (!h->singular) {
        double *U = (double *)calloc((size_t)(n * n), sizeof(double));
        int ok = 1;
        for (i64 j = 0; j < n && ok; j++) {
            double s = D[j * n + j];
            for (i64 k = 0; k < j; k++) s -= U[k * n + j] * U[k * n + j];
            if (!(s > 0.0)) { ok = 0; break; }
            double d = sqrt(s);
            U[j * n + j] = d;
            for (i64 i = j + 1; i < n; i++) {
                double t = D[j * n + i];
                for (i64 k = 0; k < j; k++) t -= U[k * n + j] * U[k * n + i];
                U[j * n + i] = t / d;
            }
        }
        if (ok) { h->coarse_mode = 1; h->cfac = U; free(D); return; }
        free(U);
    }
    double *V = (double *)malloc(sizeof(double) * (size_t)(n * n)), *w = (double *)malloc(sizeof(double) * (size_t)n);
    jacobi_eigh(n, D, V, w);
    double lmax = -INFINITY;
    for (i64 i = 0; i < n; i++) if (w[i] > lmax) lmax = w[i];
    double cut = 1e-12 * (lmax > 0 ? lmax : 0.0);
    double *P = (double *)calloc((size_t)(n * n), sizeof(double));
    for (i64 k = 0; k < n; k++) {
        if (!(w[k] > cut)) continue;
        double inv = 1.0 / w[k];
        for (i64 i = 0; i < n; i++) for (i64 j = 0; j < n; j++) P[i * n + j] += V[i * n + k] * inv * V[j * n + k];
    }
    h->coarse_mode = 2;
    h->cfac = P;
    free(D); free(V); free(w);
}

static void coarse_solve(const orc_hier *h, const double *b, double *x) {
    i64 n = h->cn;
    if (h->coarse_mode == 0) return;
    if (h->coarse_mode == 1) {
        const double *U = h->cfac;
        for (i64 i = 0; i < n; i++) { /* U^T y = b */
            double s = b[i];
            for (i64 k = 0; k < i; k++) s -= U[k * n + i] * x[k];
            x[i] = s / U[i * n + i];
        }
        for (i64 i = n - 1; i >= 0; i--) { /* U x = y */
            double s = x[i];
            for (i64 k = i + 1; k < n; k++) s -= U[i * n + k] * x[k];
            x[i] = s / U[i * n + i];
        }
    } else {
        for (i64 i = 0; i < n; i++) {
            double s = 0.0;
            for (i64 j = 0; j < n; j++) s += h->cfac[i * n + j] * b[j];
            x[i] = s;
        }
    }
}

static void level_take(orc_level *L, i64 n, i64 *ip, i64 *ix, double *a) {
    memset(L, 0, sizeof *L);
    L->n = n; L->nnz = ip[n]; L->ip = ip; L->ix = ix; L->a = a;
}
static i64 *dup_i64(const i64 *v, i64 m) {
    i64 *o = (i64 *)malloc(sizeof(i64) * (size_t)(m ? m : 1));
    memcpy(o, v, sizeof(i64) * (size_t)m);
    return o;
}
static double *dup_f64(const double *v, i64 m) {
    double *o = (double *)malloc(sizeof(double) * (size_t)(m ? m : 1));
    memcpy(o, v, sizeof(double) * (size_t)m);
    return o;
}

void orc_hier_free(orc_hier *h) {
    if (!h) return;
    for (int l = 0; l < h->nlev; l++) {
        orc_level *L = &h->lev[l];
        free(L->ip); free(L->ix); free(L->a); free(L->v2a); free(L->seeds); free(L->mptr); free(L->mem);
    }
    free(h->cfac);
    free(h);
}

/* U/hierarchy.py:120-153.  singular: -1 auto-detect, 0/1 forced.
 * Returns NULL and sets the error string on SetupError/AggregationError. */
orc_hier *orc_setup(i64 n, const i64 *ip, const i64 *ix, const double *a, u64 seed, i64 max_passes,
                    i64 cap, int passes_per_level, i64 n0, int max_levels, int singular) {
    orc_hier *h = (orc_hier *)calloc(1, sizeof(orc_hier));
    h->singular = singular < 0 ? detect_singular(n, ip, ix, a) : singular;
    i64 *cip = dup_i64(ip, n + 1), *cix = dup_i64(ix, ip[n]);
    double *ca = dup_f64(a, ip[n]);
    i64 cn = n;
    if (max_levels > 63) max_levels = 63;
    while (cn > n0 && h->nlev < max_levels - 1) {
        orc_level *L = &h->lev[h->nlev];
        level_take(L, cn, cip, cix, ca);
        i64 *v2a = (i64 *)malloc(sizeof(i64) * (size_t)cn), *seeds = (i64 *)malloc(sizeof(i64) * (size_t)cn);
        i64 nc = orc_aggregate(cn, cip, cix, ca, seed, max_passes, cap, v2a, seeds, NULL);
        if (nc < 0) { free(v2a); free(seeds); h->nlev++; orc_hier_free(h); return NULL; }
        if (passes_per_level == 2) {
            /* aggregate o galerkin o aggregate, composed (U/hierarchy.py:135-138,
             * U/aggregation.py:206-216) */
            i64 *mp, *mx; double *mv;
            orc_galerkin(cn, cip, cix, ca, v2a, nc, &mp, &mx, &mv);
            i64 *v2b = (i64 *)malloc(sizeof(i64) * (size_t)nc), *sb = (i64 *)malloc(sizeof(i64) * (size_t)nc);
            i64 nc2 = orc_aggregate(nc, mp, mx, mv, seed, max_passes, cap, v2b, sb, NULL);
            free(mp); free(mx); free(mv);
            if (nc2 < 0) { free(v2a); free(seeds); free(v2b); free(sb); h->nlev++; orc_hier_free(h); return NULL; }
            for (i64 i = 0; i < cn; i++) v2a[i] = v2b[v2a[i]];
            for (i64 I = 0; I < nc2; I++) sb[I] = seeds[sb[I]];
            memcpy(seeds, sb, sizeof(i64) * (size_t)nc2);
            nc = nc2;
            free(v2b); free(sb);
        }
        L->v2a = v2a; L->seeds = seeds; L->nc = nc;
        h->nlev++;
        if (nc == cn) {
            snprintf(g_err, sizeof g_err, "aggregation stagnated at level %d: %lld vertices produced no coarsening",
                     h->nlev - 1, (long long)cn);
            orc_hier_free(h);
            return NULL;
        }
        build_members(L);
        i64 *np_, *nx; double *nv;
        orc_galerkin(cn, cip, cix, ca, v2a, nc, &np_, &nx, &nv);
        cip = np_; cix = nx; ca = nv; cn = nc;
    }
    level_take(&h->lev[h->nlev], cn, cip, cix, ca);
    h->nlev++;
    coarse_factor(h);
    return h;
}

int orc_hier_nlevels(const orc_hier *h) { return h->nlev; }
int orc_hier_singular(const orc_hier *h) { return h->singular; }
void orc_hier_level(const orc_hier *h, int l, i64 *n, i64 *nnz, i64 *nc, const i64 **ip, const i64 **ix,
                    const double **a, const i64 **v2a, const i64 **seeds) {
    const orc_level *L = &h->lev[l];
    *n = L->n; *nnz = L->nnz; *nc = L->nc; *ip = L->ip; *ix = L->ix; *a = L->a; *v2a = L->v2a; *seeds = L->seeds;
}
void orc_coarse_solve(const orc_hier *h, const double *b, double *x) { coarse_solve(h, b, x); }

/* ------------------------------------------------------------------ */
/* solve  (U/solvers.py)                                                */
/* ------------------------------------------------------------------ */
typedef struct {
    int kcycle;          /* CycleSpec.kind == "kcycle" (U/solvers.py:39-50) */
    int inner_steps, pre, post;
    int l1;              /* Smoother.kind == "l1" (U/solvers.py:24-36) */
    double omega;
} orc_params;

static double dot(i64 n, const double *x, const double *y) {
    double s = 0.0;
    for (i64 i = 0; i < n; i++) s += x[i] * y[i];
    return s;
}
static double nrm2(i64 n, const double *x) { return sqrt(dot(n, x, x)); }
static void project_mean(i64 n, double *v) { /* U/solvers.py:112-113 */
    if (n == 0) return;
    double s = 0.0;
    for (i64 i = 0; i < n; i++) s += v[i];
    double m = s / (double)n;
    for (i64 i = 0; i < n; i++) v[i] = v[i] - m;
}
static int g_solve_err;

/* U/solvers.py:116-125 */
static void check_compatible(i64 n, double *b, int level) {
    double nb = nrm2(n, b);
    if (nb == 0.0) return;
    double s = 0.0;
    for (i64 i = 0; i < n; i++) s += b[i];
    double drift = fabs(s) / (sqrt((double)n) * nb);
    if (drift > 1e-10) {
        if (level < 0) snprintf(g_err, sizeof g_err, "right-hand side at the finest level has a null-space component (relative size %.2e > 1e-10)", drift);
        else snprintf(g_err, sizeof g_err, "right-hand side at level %d has a null-space component (relative size %.2e > 1e-10)", level, drift);
        g_solve_err = 1;
        return;
    }
    project_mean(n, b);
}

/* U/solvers.py:69-81 */
static double *inverse_diag(const orc_level *L, const orc_params *p) {
    double *m = (double *)malloc(sizeof(double) * (size_t)(L->n ? L->n : 1));
    double scale;
    if (p->l1) { orc_l1_diag(L->n, L->ip, L->ix, L->a, m); scale = 1.0; }
    else { orc_diag_of(L->n, L->ip, L->ix, L->a, m); scale = p->omega; }
    for (i64 i = 0; i < L->n; i++) {
        if (m[i] <= 0) {
            snprintf(g_err, sizeof g_err, "non-positive smoother diagonal at row %lld", (long long)i);
            g_solve_err = 1;
            free(m);
            return NULL;
        }
    }
    for (i64 i = 0; i < L->n; i++) m[i] = scale / m[i];
    return m;
}

static double *g_invm[64];

static void cycle_rec(const orc_hier *h, const orc_params *p, int l, const double *bin, double *x);

/* U/solvers.py:160-187 */
static void inner_fcg(const orc_hier *h, const orc_params *p, int l, const double *b, double *x) {
    const orc_level *L = &h->lev[l];
    i64 n = L->n;
    double *r = dup_f64(b, n), *z = (double *)malloc(sizeof(double) * (size_t)(n ? n : 1));
    double *pp = (double *)malloc(sizeof(double) * (size_t)(n ? n : 1));
    double *ap = (double *)malloc(sizeof(double) * (size_t)(n ? n : 1));
    double *pprev = (double *)malloc(sizeof(double) * (size_t)(n ? n : 1));
    double *apprev = (double *)malloc(sizeof(double) * (size_t)(n ? n : 1));
    int have_prev = 0;
    for (i64 i = 0; i < n; i++) x[i] = 0.0;
    double bn = nrm2(n, b);
    for (int k = 0; k < p->inner_steps; k++) {
        if (nrm2(n, r) <= 1e-14 * bn) break;
        cycle_rec(h, p, l, r, z);
        if (g_solve_err) break;
        if (!have_prev) memcpy(pp, z, sizeof(double) * (size_t)n);
        else {
            double beta = -dot(n, z, apprev) / dot(n, pprev, apprev);
            for (i64 i = 0; i < n; i++) pp[i] = z[i] + beta * pprev[i];
        }
        orc_spmv(n, L->ip, L->ix, L->a, pp, ap);
        double pap = dot(n, pp, ap);
        if (pap <= 0.0) break;
        double alpha = dot(n, pp, r) / pap;
        for (i64 i = 0; i < n; i++) x[i] = x[i] + alpha * pp[i];
        for (i64 i = 0; i < n; i++) r[i] = r[i] - alpha * ap[i];
        if (h->singular) project_mean(n, r);
        memcpy(pprev, pp, sizeof(double) * (size_t)n);
        memcpy(apprev, ap, sizeof(double) * (size_t)n);
        have_prev = 1;
    }
    free(r); free(z); free(pp); free(ap); free(pprev); free(apprev);
}

/* U/solvers.py:128-157 */
static void cycle_rec(const orc_hier *h, const orc_params *p, int l, const double *bin, double *x) {
    const orc_level *L = &h->lev[l];
    i64 n = L->n;
    double *b = dup_f64(bin, n);
    if (h->singular) { check_compatible(n, b, l); if (g_solve_err) { free(b); return; } }
    if (l == h->nlev - 1) {
        coarse_solve(h, b, x);
        if (h->singular) project_mean(n, x);
        free(b);
        return;
    }
    double *r = (double *)malloc(sizeof(double) * (size_t)n);
    for (i64 i = 0; i < n; i++) x[i] = 0.0;
    orc_smooth_sweeps(n, L->ip, L->ix, L->a, g_invm[l], x, b, p->pre, r);
    orc_spmv(n, L->ip, L->ix, L->a, x, r);
    for (i64 i = 0; i < n; i++) r[i] = b[i] - r[i];
    i64 nc = L->nc;
    double *rc = (double *)malloc(sizeof(double) * (size_t)(nc ? nc : 1)), *ec = (double *)malloc(sizeof(double) * (size_t)(nc ? nc : 1));
    orc_restrict(nc, L->mptr, L->mem, r, rc);
    if (h->singular) project_mean(nc, rc);
    int exact = (l + 1 == h->nlev - 1);
    if (!p->kcycle || p->inner_steps == 0 || exact) cycle_rec(h, p, l + 1, rc, ec);
    else inner_fcg(h, p, l + 1, rc, ec);
    if (!g_solve_err) {
        for (i64 i = 0; i < n; i++) x[i] = x[i] + ec[L->v2a[i]];
        orc_smooth_sweeps(n, L->ip, L->ix, L->a, g_invm[l], x, b, p->post, r);
        if (h->singular) project_mean(n, x);
    }
    free(b); free(r); free(rc); free(ec);
}

/* U/solvers.py:190-255.  Returns 0 ok, 1 NumericalError (message in
 * orc_last_error; history/iterations filled up to the failure), 2 ValueError.
 * history must hold max_iters+1 entries. */
int orc_npcg_solve(const orc_hier *h, int kcycle, int inner_steps, int pre, int post, int l1, double omega,
                   const double *bin, double tol, i64 max_iters, const double *x0, double *x_out,
                   double *history, i64 *iterations, int *converged) {
    orc_params P = {kcycle, inner_steps, pre, post, l1, omega};
    g_solve_err = 0;
    if (tol <= 0) { set_err("tol must be positive"); return 2; }
    const orc_level *L = &h->lev[0];
    i64 n = L->n;
    for (int l = 0; l < h->nlev; l++) g_invm[l] = NULL;
    double *b = dup_f64(bin, n);
    *iterations = 0; *converged = 0;
    if (h->singular) { check_compatible(n, b, -1); if (g_solve_err) { free(b); return 1; } }
    double bn = nrm2(n, b);
    if (bn == 0.0) {
        for (i64 i = 0; i < n; i++) x_out[i] = 0.0;
        history[0] = 0.0; *converged = 1; free(b);
        return 0;
    }
    for (int l = 0; l < h->nlev - 1; l++) {
        g_invm[l] = inverse_diag(&h->lev[l], &P);
        if (g_solve_err) { free(b); return 1; }
    }
    double *x = x_out, *r = (double *)malloc(sizeof(double) * (size_t)n);
    double *z = (double *)malloc(sizeof(double) * (size_t)n), *pp = (double *)malloc(sizeof(double) * (size_t)n);
    double *ap = (double *)malloc(sizeof(double) * (size_t)n), *pprev = (double *)malloc(sizeof(double) * (size_t)n);
    double *apprev = (double *)malloc(sizeof(double) * (size_t)n);
    if (!x0) { for (i64 i = 0; i < n; i++) x[i] = 0.0; memcpy(r, b, sizeof(double) * (size_t)n); }
    else {
        memcpy(x, x0, sizeof(double) * (size_t)n);
        if (h->singular) project_mean(n, x);
        orc_spmv(n, L->ip, L->ix, L->a, x, r);
        for (i64 i = 0; i < n; i++) r[i] = b[i] - r[i];
    }
    i64 nh = 0;
    history[nh++] = nrm2(n, r) / bn;
    int have_prev = 0, up = 0, rc = 0;
    i64 it = 0;
    while (history[nh - 1] > tol && it < max_iters) {
        cycle_rec(h, &P, 0, r, z);
        if (g_solve_err) { rc = 1; break; }
        if (h->singular) project_mean(n, z);
        if (!have_prev) memcpy(pp, z, sizeof(double) * (size_t)n);
        else {
            double beta = -dot(n, z, apprev) / dot(n, pprev, apprev);
            for (i64 i = 0; i < n; i++) pp[i] = z[i] + beta * pprev[i];
        }
        orc_spmv(n, L->ip, L->ix, L->a, pp, ap);
        double pap = dot(n, pp, ap);
        if (pap <= 0.0) {
            snprintf(g_err, sizeof g_err, "conjugate-gradient breakdown at iteration %lld: p'Ap = %.3e",
                     (long long)(it + 1), pap);
            rc = 1;
            break;
        }
        double alpha = dot(n, pp, r) / pap;
        for (i64 i = 0; i < n; i++) x[i] = x[i] + alpha * pp[i];
        for (i64 i = 0; i < n; i++) r[i] = r[i] - alpha * ap[i];
        if (h->singular) { project_mean(n, r); project_mean(n, x); }
        double rel = nrm2(n, r) / bn;
        history[nh++] = rel;
        it++;
        if (rel > history[nh - 2]) up++; else up = 0;
        if (up >= 2) { have_prev = 0; up = 0; }
        else {
            memcpy(pprev, pp, sizeof(double) * (size_t)n);
            memcpy(apprev, ap, sizeof(double) * (size_t)n);
            have_prev = 1;
        }
    }
    *iterations = it;
    *converged = history[nh - 1] <= tol;
    for (int l = 0; l < h->nlev; l++) { free(g_invm[l]); g_invm[l] = NULL; }
    free(b); free(r); free(z); free(pp); free(ap); free(pprev); free(apprev);
    return rc;
}
