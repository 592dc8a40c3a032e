// kernels_setup.cu -- setup-phase kernels: counter hash + quasi-random
// scores, distance-3 MIS selection and claim as two max-hops over A (no A^2),
// conflict-free aggregate admission, renumbering by ascending seed,
// members_csr, Galerkin coarse operator as an exact-order segmented
// sum-by-aggregate-pair, dense coarsest factorization.
//
// Reference: U/aggregation.py:130-203, U/hierarchy.py:22-65,
// K/numba_backend.py:14-44 (hash), :100-111 (scores), :145-273.
#include <cooperative_groups.h>
#include <chrono>
#include <cstring>
#include <cub/cub.cuh>

#include "setup.h"

namespace cg = cooperative_groups;

namespace uaamg {

// ============================================================ hash + scores
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t pass_base(uint64_t seed, int64_t pass_idx) {
    uint64_t z = seed ^ (0xA0761D6478BD642Full * (uint64_t)(pass_idx + 1));
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ double hash_unit(uint64_t base, int64_t i) {
    const uint64_t z = mix64(mix64(base + (uint64_t)i * 0x9E3779B97F4A7C15ull));
    return __dmul_rn((double)(z >> 11), 1.0 / 9007199254740992.0);
}

__global__ void k_hash_u01(uint64_t base, const int64_t* idx, int64_t m, double* out) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x)
        out[k] = hash_unit(base, idx[k]);
}
void launch_hash_u01(uint64_t seed, int64_t pass_idx, const int64_t* idx, int64_t m, double* out, cudaStream_t s) {
    if (m == 0) return;
    UA_LAUNCH(k_hash_u01, cdiv(m, 256) > 4096 ? 4096 : cdiv(m, 256), 256, 0, s, pass_base(seed, pass_idx), idx, m,
              out);
}

// structural off-diagonal count (K/numba_backend.py:87-97)
__global__ void k_degrees(Csr A, int* deg) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += gridDim.x * blockDim.x) {
        int d = 0;
        for (int k = A.rp[i]; k < A.rp[i + 1]; ++k) d += (A.ci[k] != i);
        deg[i] = d;
    }
}
void launch_degrees(const Csr& A, int* deg, cudaStream_t s) {
    UA_LAUNCH(k_degrees, cdiv(A.n, 256), 256, 0, s, A, deg);
}

// v_i = d_i + ((i mod 12) + u_i) / 12, in exactly that evaluation order
// (K/numba_backend.py:110)
__global__ void k_scores(int n, const int* deg, uint64_t base, double* s) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double u = hash_unit(base, i);
        s[i] = __dadd_rn((double)deg[i], __ddiv_rn(__dadd_rn((double)(i % 12), u), 12.0));
    }
}
void launch_scores(const Csr& A, const int* deg, uint64_t seed, int64_t pass_idx, double* scores, cudaStream_t s) {
    UA_LAUNCH(k_scores, cdiv(A.n, 256), 256, 0, s, A.n, deg, pass_base(seed, pass_idx), scores);
}

// ============================================================ MIS / claim hops
// key(j) = (s_j, -j): j beats i iff s_j > s_i or (s_j == s_i and j < i)
__device__ __forceinline__ bool key_gt(double sa, int ia, double sb, int ib) {
    return sa > sb || (sa == sb && ia < ib);
}

// vertex state: 0 unprocessed, 1 center of the current pass, 2 processed
// hop 1: m[k] = max key over j in row k with (mode 0: state != 2, mode 1: state == 1)
__global__ void k_hop1(Csr A, const double* __restrict__ s, const uint8_t* __restrict__ st, int mode,
                       double* __restrict__ ms, int* __restrict__ mi) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < A.n; k += gridDim.x * blockDim.x) {
        double bs = 0.0;
        int bi = -1;
        for (int e = A.rp[k]; e < A.rp[k + 1]; ++e) {
            const int j = __ldg(A.ci + e);
            const uint8_t sj = __ldg(st + j);
            if (mode == 0 ? (sj == 2) : (sj != 1)) continue;
            const double v = __ldg(s + j);
            if (bi < 0 || key_gt(v, j, bs, bi)) { bs = v; bi = j; }
        }
        ms[k] = bs;
        mi[k] = bi;
    }
}

// hop 2, selection (K/numba_backend.py:175-193): unprocessed i is a center
// iff no unprocessed j != i within distance 2 has a larger key.
__global__ void k_select(Csr A, const double* __restrict__ s, uint8_t* st, const double* __restrict__ ms,
                         const int* __restrict__ mi, int* n_centers) {
    int local = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += gridDim.x * blockDim.x) {
        if (st[i] != 0) continue;
        double bs = 0.0;
        int bi = -1;
        for (int e = A.rp[i]; e < A.rp[i + 1]; ++e) {
            const int k = __ldg(A.ci + e);
            const int c = __ldg(mi + k);
            if (c < 0) continue;
            const double v = __ldg(ms + k);
            if (bi < 0 || key_gt(v, c, bs, bi)) { bs = v; bi = c; }
        }
        const double si = s[i];
        if (bi < 0 || bi == i || key_gt(si, i, bs, bi)) {
            st[i] = 1;
            ++local;
        }
    }
    local = __reduce_add_sync(0xffffffffu, local);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(n_centers, local);
}

// hop 2, claim (K/numba_backend.py:196-220): owner = best center within
// distance 2 if its score >= own score, centers own themselves.
__global__ void k_claim(Csr A, const double* __restrict__ s, const uint8_t* __restrict__ st,
                        const double* __restrict__ ms, const int* __restrict__ mi, int* owner) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < A.n; j += gridDim.x * blockDim.x) {
        const uint8_t sj = st[j];
        if (sj == 1) { owner[j] = j; continue; }
        if (sj == 2) { owner[j] = -1; continue; }
        double bs = 0.0;
        int bi = -1;
        for (int e = A.rp[j]; e < A.rp[j + 1]; ++e) {
            const int k = __ldg(A.ci + e);
            const int c = __ldg(mi + k);
            if (c < 0) continue;
            const double v = __ldg(ms + k);
            if (bi < 0 || key_gt(v, c, bs, bi)) { bs = v; bi = c; }
        }
        owner[j] = (bi >= 0 && !(bs < s[j])) ? bi : -1;
    }
}

// explicit-pattern variants (kernel table: pattern = A^2)
__global__ void k_select_pattern(Csr P, const double* s, const uint8_t* processed, uint8_t* out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n; i += gridDim.x * blockDim.x) {
        if (processed[i]) { out[i] = 0; continue; }
        bool ok = true;
        const double si = s[i];
        for (int e = P.rp[i]; e < P.rp[i + 1]; ++e) {
            const int j = P.ci[e];
            if (j == i || processed[j]) continue;
            if (!key_gt(si, i, s[j], j)) { ok = false; break; }
        }
        out[i] = ok;
    }
}
__global__ void k_claim_pattern(Csr P, const double* s, const uint8_t* processed, const uint8_t* is_center,
                                int* owner) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < P.n; j += gridDim.x * blockDim.x) {
        if (is_center[j]) { owner[j] = j; continue; }
        owner[j] = -1;
        if (processed[j]) continue;
        int best = -1;
        double bs = 0.0;
        const double sj = s[j];
        for (int e = P.rp[j]; e < P.rp[j + 1]; ++e) {
            const int i = P.ci[e];
            if (!is_center[i]) continue;
            const double si = s[i];
            if (si < sj) continue;
            if (best == -1 || key_gt(si, i, bs, best)) { best = i; bs = si; }
        }
        owner[j] = best;
    }
}

// ============================================================ admission
// Uncapped (size_cap=None): the reference's repeated strongest-first sweeps
// (K/numba_backend.py:235-273) admit exactly the bucket vertices connected to
// the center through admitted bucket vertices, independent of sweep order.
// That fixpoint is computed here by monotone label propagation.
__global__ void k_admit_init(int n, const uint8_t* st, const int* owner, uint8_t* adm) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
        adm[j] = (st[j] == 1);
}
__global__ void k_admit_step(Csr A, const int* __restrict__ owner, uint8_t* adm, int* changed) {
    int local = 0;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < A.n; j += gridDim.x * blockDim.x) {
        const int c = owner[j];
        if (c < 0 || c == j || adm[j]) continue;
        for (int e = A.rp[j]; e < A.rp[j + 1]; ++e) {
            const int nb = __ldg(A.ci + e);
            if (((volatile uint8_t*)adm)[nb] && __ldg(owner + nb) == c) {
                adm[j] = 1;
                local = 1;
                break;
            }
        }
    }
    if (__any_sync(0xffffffffu, local) && (threadIdx.x & 31) == 0) atomicOr(changed, 1);
}
// commit: admitted vertices and centers become processed with their seed
__global__ void k_admit_commit(int n, uint8_t* st, const int* owner, const uint8_t* adm, int* seed_of,
                               int* remaining) {
    int local = 0;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const uint8_t sj = st[j];
        if (sj == 1 || (sj == 0 && adm[j])) {
            seed_of[j] = owner[j];
            st[j] = 2;
        } else if (sj == 0) {
            ++local;
        }
    }
    local = __reduce_add_sync(0xffffffffu, local);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(remaining, local);
}

// Capped: per-center sequential greedy exactly as the reference (bucket in
// ascending vertex order, candidates by descending |A_cj| stable, sweeps).
__global__ void k_bucket_count(int n, const uint8_t* st, const int* owner, int* cnt) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const int c = owner[j];
        if (c >= 0 && st[j] == 0) atomicAdd(cnt + c, 1);
    }
}
__global__ void k_bucket_fill(int n, const uint8_t* st, const int* owner, const int* bptr, int* cursor, int* bjs) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const int c = owner[j];
        if (c >= 0 && st[j] == 0) bjs[bptr[c] + atomicAdd(cursor + c, 1)] = j;
    }
}
__device__ int lower_bound_i(const int* v, int lo, int hi, int key) {
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (v[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}
// one thread per center; scratch ord/adm per bucket slot
__global__ void k_admit_capped(Csr A, int n, const uint8_t* st, const int* bptr, int* bjs, int* ord, double* w,
                               uint8_t* admf, long long cap, int* seed_of, uint8_t* newly) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
        if (st[c] != 1) continue;
        const int lo = bptr[c], m = bptr[c + 1] - lo;
        int* js = bjs + lo;
        int* od = ord + lo;
        double* wv = w + lo;
        uint8_t* ad = admf + lo;
        // ascending vertex order within the bucket (U/aggregation.py:157,164)
        for (int a = 1; a < m; ++a) {
            const int t = js[a];
            int b = a - 1;
            while (b >= 0 && js[b] > t) { js[b + 1] = js[b]; --b; }
            js[b + 1] = t;
        }
        const int rs = A.rp[c], re = A.rp[c + 1];
        for (int t = 0; t < m; ++t) {
            const int pos = lower_bound_i(A.ci, rs, re, js[t]);
            wv[t] = (pos < re && A.ci[pos] == js[t]) ? fabs(A.av[pos]) : 0.0;
            ad[t] = 0;
            // stable insertion by descending weight (mergesort of -w)
            int b = t - 1;
            while (b >= 0 && wv[od[b]] < wv[t]) { od[b + 1] = od[b]; --b; }
            od[b + 1] = t;
        }
        long long count = 1;
        bool progress = true;
        while (progress && count < cap) {
            progress = false;
            for (int t = 0; t < m; ++t) {
                if (count >= cap) break;
                const int id = od[t];
                if (ad[id]) continue;
                const int j = js[id];
                bool conn = false;
                for (int e = A.rp[j]; e < A.rp[j + 1]; ++e) {
                    const int nb = A.ci[e];
                    if (nb == c) { conn = true; break; }
                    const int pos = lower_bound_i(js, 0, m, nb);
                    if (pos < m && js[pos] == nb && ad[pos]) { conn = true; break; }
                }
                if (conn) {
                    ad[id] = 1;
                    seed_of[j] = c;
                    newly[j] = 1;
                    ++count;
                    progress = true;
                }
            }
        }
        seed_of[c] = c;
    }
}
__global__ void k_capped_commit(int n, uint8_t* st, uint8_t* newly, int* remaining) {
    int local = 0;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        if (st[j] == 1 || newly[j]) { st[j] = 2; newly[j] = 0; }
        else if (st[j] == 0) ++local;
    }
    local = __reduce_add_sync(0xffffffffu, local);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(remaining, local);
}

// ============================================================ cooperative aggregation
// The whole multi-pass PAA of one level (U/aggregation.py:184-194) in one
// cooperative launch: scores -> max-hop -> select -> max-hop -> claim ->
// admission fixpoint -> commit, separated by grid-wide barriers, with the
// pass / admission loop control read from device counters (no host round
// trips).  Pass 0 sweeps every vertex; later passes work on worklists: U =
// the still-unprocessed vertices (compacted at each commit) and H = U plus
// its neighbours (the only vertices whose hop values a selection or claim in
// U reads).  Appends are atomic, so list order varies, but every phase is
// order-free (key maxima, flags, a monotone fixpoint), so results are
// bit-identical to the full sweeps.  Processed vertices keep stale
// owner/adm values; they cannot match a current center (centers are
// unprocessed until their own commit).  Short rows are handled
// thread-per-item, rows longer than kLongRow warp-per-item from a list of
// the level's long rows (built once; membership in U / H is checked per
// item), so the warp loops cost nothing on levels without long rows.
struct AggCoop {
    Csr A;
    const int* longs;     // rows longer than kLongRow (any order)
    const int* nlongs;    // their count (device)
    const int* deg;
    uint64_t seed;
    int max_passes;
    uint8_t* st;
    double* sc;
    double* ms;
    int* mi;
    int* owner;
    uint8_t* adm;
    int* seed_of;
    int* ulist[2];  // U, double-buffered by pass parity
    int* hlist;     // H
    int* mark;      // pass stamp of H membership
    int* ctl;  // [0..2] centers / pass slot, [3..5] remaining / pass slot, [6..8] changed / iteration slot,
               // [9] passes, [10] leftover, [11..13] |U'| / pass slot, [14..15] |H| / pass parity
    unsigned long long* prof;  // diagnostics (UAAMG_AGG_PROF): per pass {t_start, |U|, |H|, admission iterations}
    const int* symc;  // k_pattern_sym: {upper entries without a mirror, upper count, lower count}
};

// Structural symmetry of A's pattern: the admission sweeps'
// shortcut (admitting j's same-owner neighbours when j is admitted) relies on
// nb in row(j) => j in row(nb); the reference only tests row(j) itself
// (K/numba_backend.py:256-266).  Warp per row: every upper entry (i, j > i)
// looks for i in row j (binary search); with every upper entry mirrored and
// as many lower as upper entries, the pattern is symmetric.
__global__ void k_pattern_sym(Csr A, int* symc) {
    const int lane = threadIdx.x & 31;
    int miss = 0, up = 0, lo = 0;
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < A.n; i += (gridDim.x * blockDim.x) >> 5) {
        const int e0 = A.rp[i], e1 = A.rp[i + 1];
        for (int e = e0 + lane; e < e1; e += 32) {
            const int j = __ldg(A.ci + e);
            if (j < i) { ++lo; continue; }
            if (j == i) continue;
            ++up;
            int a = __ldg(A.rp + j), b = __ldg(A.rp + j + 1);
            while (a < b) {
                const int m = (a + b) >> 1;
                if (__ldg(A.ci + m) < i) a = m + 1; else b = m;
            }
            if (!(a < __ldg(A.rp + j + 1) && __ldg(A.ci + a) == i)) ++miss;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        miss += __shfl_xor_sync(0xffffffffu, miss, o);
        up += __shfl_xor_sync(0xffffffffu, up, o);
        lo += __shfl_xor_sync(0xffffffffu, lo, o);
    }
    if (lane == 0 && (miss | up | lo)) {
        if (miss) atomicAdd(symc, miss);
        atomicAdd(symc + 1, up);
        atomicAdd(symc + 2, lo);
    }
}

__device__ __forceinline__ void warp_keymax(double& s, int& i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double s2 = __shfl_xor_sync(0xffffffffu, s, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, i, o);
        if (i2 >= 0 && (i < 0 || key_gt(s2, i2, s, i))) { s = s2; i = i2; }
    }
}

// max key over row r of the hop-1 table (ms, mi); lanes split the row when
// warp (step 32: four strided entries per lane in flight -- the key order is
// total, so the maximum does not depend on the visiting order)
__device__ __forceinline__ void row_hopmax(const Csr& A, const double* ms, const int* mi, int r, int e0, int e1,
                                           int step, double& bs, int& bi) {
    if (step == 1) {
        // one thread: 8 entries in flight per batch
        for (int e = e0; e < e1; e += 8) {
            int k[8], c[8];
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) k[q] = e + q < e1 ? __ldg(A.ci + e + q) : -1;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                c[q] = k[q] >= 0 ? mi[k[q]] : -1;
                v[q] = k[q] >= 0 ? ms[k[q]] : 0.0;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (c[q] >= 0 && (bi < 0 || key_gt(v[q], c[q], bs, bi))) { bs = v[q]; bi = c[q]; }
        }
        return;
    }
    for (int e = e0; e < e1; e += 4 * step) {
        int k[4], c[4];
        double v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) k[q] = e + q * step < e1 ? __ldg(A.ci + e + q * step) : -1;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            c[q] = k[q] >= 0 ? mi[k[q]] : -1;
            v[q] = k[q] >= 0 ? ms[k[q]] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (c[q] >= 0 && (bi < 0 || key_gt(v[q], c[q], bs, bi))) { bs = v[q]; bi = c[q]; }
    }
}

// items [0, cnt) of a worklist (list == nullptr: the identity, all vertices)
struct WL {
    const int* list;
    int cnt;
    __device__ __forceinline__ int operator[](int t) const { return list ? list[t] : t; }
};

// Long rows (> kLongRow entries) of a phase: `team` warps of one CTA per row
// (team = the power of two that spreads the level's long rows over the whole
// grid, up to the CTA), so a hub row of thousands of entries is not one
// warp's serial chain of dependent gathers.  filt(k): whether row k takes
// part (evaluated identically by every warp of its team); part(k, e, e1,
// step, bs, bi): key maximum over entries e, e + step, ... < e1; fin(k, bs,
// bi): the row's result, called by one thread.  The key order is total, so
// the split does not change any maximum.  Iterations are CTA-uniform, so
// __syncthreads joins a team's warps.
__device__ __forceinline__ int long_team(int nlong, int nw) {
    const int W = blockDim.x >> 5;
    if (nlong <= 0) return 1;
    int t = 1;
    while (2 * t <= W && 2 * t * nlong <= nw) t *= 2;
    return t;
}
template <class Filt, class Part, class Fin>
__device__ __forceinline__ void agg_long(const AggCoop& g, int nlong, int team, int lane, int w, int nw, Filt filt,
                                         Part part, Fin fin) {
    const Csr& A = g.A;
    if (team <= 1) {
        for (int t = w; t < nlong; t += nw) {
            const int k = g.longs[t];
            if (!filt(k)) continue;
            double bs = 0.0;
            int bi = -1;
            part(k, A.rp[k] + lane, A.rp[k + 1], 32, bs, bi);
            warp_keymax(bs, bi);
            if (lane == 0) fin(k, bs, bi);
        }
        return;
    }
    __shared__ double tbs[32];
    __shared__ int tbi[32];
    const int wib = threadIdx.x >> 5, tpb = (blockDim.x >> 5) / team;
    for (int base = blockIdx.x * tpb; base < nlong; base += gridDim.x * tpb) {
        const int li = base + wib / team;
        double bs = 0.0;
        int bi = -1;
        int k = -1;
        if (li < nlong) {
            k = g.longs[li];
            if (filt(k))
                part(k, A.rp[k] + (wib % team) * 32 + lane, A.rp[k + 1], 32 * team, bs, bi);
            else
                k = -1;
        }
        warp_keymax(bs, bi);
        if (lane == 0) {
            tbs[wib] = bs;
            tbi[wib] = bi;
        }
        __syncthreads();
        if (k >= 0 && wib % team == 0 && lane == 0) {
            for (int q = 1; q < team; ++q) {
                const double s2 = tbs[wib + q];
                const int i2 = tbi[wib + q];
                if (i2 >= 0 && (bi < 0 || key_gt(s2, i2, bs, bi))) { bs = s2; bi = i2; }
            }
            fin(k, bs, bi);
        }
        __syncthreads();
    }
}

// hop1 over the items of H: max key over the row's unprocessed (mode 0) or
// center (mode 1) neighbours
__device__ void coop_hop1(const AggCoop& g, WL H, int mode, int stamp, int nlong, int tid, int nth, int lane, int w,
                          int nw) {
    const Csr& A = g.A;
    for (int t = tid; t < H.cnt; t += nth) {
        const int k = H[t];
        const int e0 = A.rp[k], e1 = A.rp[k + 1];
        if (e1 - e0 > kLongRow) continue;
        double bs = 0.0;
        int bi = -1;
        for (int e = e0; e < e1; e += 8) {
            int j[8];
            uint8_t sj[8];
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) j[q] = e + q < e1 ? __ldg(A.ci + e + q) : -1;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                sj[q] = j[q] >= 0 ? g.st[j[q]] : (mode == 0 ? 2 : 0);  // padding: skipped
                v[q] = j[q] >= 0 ? g.sc[j[q]] : 0.0;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (mode == 0 ? (sj[q] == 2) : (sj[q] != 1)) continue;
                if (bi < 0 || key_gt(v[q], j[q], bs, bi)) { bs = v[q]; bi = j[q]; }
            }
        }
        g.ms[k] = bs;
        g.mi[k] = bi;
    }
    agg_long(
        g, nlong, long_team(nlong, nw), lane, w, nw, [&](int k) { return !H.list || g.mark[k] == stamp; },
        [&](int, int e, int e1, int step, double& bs, int& bi) {
            for (; e < e1; e += 4 * step) {
                int j[4];
                uint8_t sj[4];
                double v[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) j[q] = e + step * q < e1 ? __ldg(A.ci + e + step * q) : -1;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    sj[q] = j[q] >= 0 ? g.st[j[q]] : (mode == 0 ? 2 : 0);  // padding: skipped
                    v[q] = j[q] >= 0 ? g.sc[j[q]] : 0.0;
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (mode == 0 ? (sj[q] == 2) : (sj[q] != 1)) continue;
                    if (bi < 0 || key_gt(v[q], j[q], bs, bi)) { bs = v[q]; bi = j[q]; }
                }
            }
        },
        [&](int k, double bs, int bi) {
            g.ms[k] = bs;
            g.mi[k] = bi;
        });
}

// block-aggregated compaction: each thread tests 4 consecutive vertices, a
// block scan places them and ONE atomic per block tile reserves the range
// (one atomic per warp was ~65K same-address atomics at level 0, ~45 us)
// items t in [0, m): f(t, v) says whether to append v (called once per item)
template <class F>
__device__ void wl_compact_blk(int m, F f, int* list, int* cnt) {
    __shared__ int wsum[32];
    __shared__ int bbase;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nwb = blockDim.x >> 5;
    const int tile = blockDim.x * 4;
    for (int base = blockIdx.x * tile; base < m; base += gridDim.x * tile) {
        const int k0 = base + threadIdx.x * 4;
        unsigned bits = 0;
        int vals[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (k0 + q < m && f(k0 + q, vals[q])) bits |= 1u << q;
        const int c = __popc(bits);
        int x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[wib] = x;
        __syncthreads();
        if (wib == 0) {
            int v = lane < nwb ? wsum[lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += y;
            }
            if (lane < nwb) wsum[lane] = v;  // inclusive
            const int tot = __shfl_sync(0xffffffffu, v, 31);
            if (lane == 0) bbase = tot ? atomicAdd(cnt, tot) : 0;
        }
        __syncthreads();
        int off = bbase + (wib ? wsum[wib - 1] : 0) + x - c;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (bits >> q & 1u) list[off++] = vals[q];
        __syncthreads();
    }
}
__device__ void wl_compact(const int* mark, int stamp, int n, int* list, int* cnt, int, int) {
    wl_compact_blk(n, [&](int k, int& v) { v = k; return mark[k] == stamp; }, list, cnt);
}
__device__ void wl_compact_st(const uint8_t* st, int n, int* list, int* cnt, int, int) {
    wl_compact_blk(n, [&](int k, int& v) { v = k; return st[k] == 0; }, list, cnt);
}

// rows longer than kLongRow, appended in any order
__global__ void k_long_rows(Csr A, int* list, int* cnt) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += gridDim.x * blockDim.x)
        if (A.rp[i + 1] - A.rp[i] > kLongRow) list[atomicAdd(cnt, 1)] = i;
}

// barrier between phases: the whole cooperative grid, or -- small levels --
// one thread-block cluster (hardware barrier, release/acquire at cluster
// scope; the acquire invalidates L1, so plain loads see the other CTAs'
// global writes)
// Grid barrier on a monotonic arrival counter (ctl[20], zeroed per launch):
// thread 0 of each CTA adds with release semantics, spins with relaxed loads
// until every CTA of this epoch has arrived, then fences once (acquire; it
// also invalidates L1, so plain loads after the barrier see other CTAs'
// writes).
// No last-arriver round trip and no full fences: ~1 us cheaper per phase
// than cg::grid_group::sync().  A lost CTA traps instead of hanging.
struct GridBar {
    unsigned* cnt = nullptr;
    unsigned ep = 0;
    __device__ void init(int* ctl) { cnt = reinterpret_cast<unsigned*>(ctl + 20); }
    __device__ void sync() {
        __syncthreads();
        ++ep;
        if (threadIdx.x == 0) {
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
            const unsigned target = ep * gridDim.x;
            const long long t0 = clock64();
            unsigned v;
            while (true) {
                asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
                if ((int)(v - target) >= 0) break;
                if (clock64() - t0 > (1ll << 34)) __trap();
            }
            asm volatile("fence.acq_rel.gpu;" ::: "memory");  // one acquire after the relaxed spin
        }
        __syncthreads();
    }
};
struct GridBarCg {  // A/B reference (UAAMG_AGG_CG_SYNC)
    __device__ void init(int*) {}
    __device__ void sync() const { cg::this_grid().sync(); }
};
struct ClusterBar {
    __device__ void init(int*) {}
    __device__ void sync() const {
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
};
constexpr int kAggClusterThreads = 1024;
constexpr int kAggClusterCtas = 16;
constexpr int kAggClusterMaxRows = 32768;  // levels up to this size aggregate on one cluster (measured: C2 L2, 42404 rows, faster on the grid)

// UAAMG_AGG_PROF: globaltimer after each phase barrier of passes 0-1
#define AGG_STAMP(K)                                                          \
    if (g.prof && pass < 2 && tid == 0) {                                     \
        unsigned long long tt;                                                \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));                \
        g.prof[140 + pass * 16 + (K)] = tt;                                   \
    }
template <class Bar>
__device__ __forceinline__ void k_aggregate_body(const AggCoop& g) {
    Bar grid{};
    grid.init(g.ctl);
    const Csr& A = g.A;
    const int n = A.n;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31, w = tid >> 5, nw = nth >> 5;
    volatile int* ctl = g.ctl;
    int remaining = n, pass = 0, itg = 0;
    const int nlong = *g.nlongs;
    WL U{nullptr, n}, H{nullptr, n};
    for (; pass < g.max_passes; ++pass) {
        if (remaining == 0) break;  // U/aggregation.py:186
        const int ps = pass % 3;
        int* unext = g.ulist[(pass + 1) & 1];
        if (tid == 0) {
            ctl[(pass + 1) % 3] = 0;
            ctl[3 + (pass + 1) % 3] = 0;
            ctl[11 + (pass + 1) % 3] = 0;
            ctl[14 + ((pass + 1) & 1)] = 0;
        }
        if (g.prof && tid == 0 && pass < 32) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
            g.prof[4 * pass] = t;
            g.prof[4 * pass + 1] = U.cnt;
        }
        const int itg0 = itg;
        // scores of U (K/numba_backend.py:100-111); mark H = U and its
        // neighbours (plain stores), then compact H in vertex order
        const uint64_t base = pass_base(g.seed, pass);
        const int stamp = pass + 1;
        int* hcnt = (int*)&ctl[14 + (pass & 1)];
        for (int t = tid; t < U.cnt; t += nth) {
            const int i = U[t];
            const double u = hash_unit(base, i);
            g.sc[i] = __dadd_rn((double)g.deg[i], __ddiv_rn(__dadd_rn((double)(i % 12), u), 12.0));
            if (U.list) {
                g.mark[i] = stamp;
                for (int e = A.rp[i]; e < A.rp[i + 1]; ++e) g.mark[__ldg(A.ci + e)] = stamp;
            }
        }
        grid.sync();
        AGG_STAMP(0);
        if (U.list) {
            wl_compact(g.mark, stamp, n, g.hlist, hcnt, tid, nth);
            grid.sync();
            AGG_STAMP(1);
            H = WL{g.hlist, ctl[14 + (pass & 1)]};
        }
        coop_hop1(g, H, 0, stamp, nlong, tid, nth, lane, w, nw);
        grid.sync();
        AGG_STAMP(2);
        // selection (K/numba_backend.py:175-193)
        int local = 0;
        for (int t = tid; t < U.cnt; t += nth) {
            const int i = U[t];
            const int e0 = A.rp[i], e1 = A.rp[i + 1];
            if (e1 - e0 > kLongRow || g.st[i] != 0) continue;
            double bs = 0.0;
            int bi = -1;
            row_hopmax(A, g.ms, g.mi, i, e0, e1, 1, bs, bi);
            if (bi < 0 || bi == i || key_gt(g.sc[i], i, bs, bi)) { g.st[i] = 1; ++local; }
        }
        const int team = long_team(nlong, nw);
        auto hopmax = [&](int k, int e, int e1, int step, double& bs, int& bi) {
            row_hopmax(A, g.ms, g.mi, k, e, e1, step, bs, bi);
        };
        agg_long(
            g, nlong, team, lane, w, nw, [&](int i) { return g.st[i] == 0; }, hopmax,  // in U, not yet a center
            [&](int i, double bs, int bi) {
                if (bi < 0 || bi == i || key_gt(g.sc[i], i, bs, bi)) { g.st[i] = 1; ++local; }
            });
        // one atomic per warp: per-thread same-address atomics serialise in L2
        // (~300K of them at level 0 cost ~100 us per phase)
        local = __reduce_add_sync(0xffffffffu, local);
        if (lane == 0 && local) atomicAdd((int*)&ctl[ps], local);
        grid.sync();
        AGG_STAMP(3);
        coop_hop1(g, H, 1, stamp, nlong, tid, nth, lane, w, nw);
        grid.sync();
        AGG_STAMP(4);
        // claim (K/numba_backend.py:196-220) + admission seeds
        for (int t = tid; t < U.cnt; t += nth) {
            const int j = U[t];
            const int e0 = A.rp[j], e1 = A.rp[j + 1];
            const uint8_t sj = g.st[j];
            g.adm[j] = (sj == 1);
            if (sj == 1) { g.owner[j] = j; continue; }
            if (sj == 2) { g.owner[j] = -1; continue; }
            if (e1 - e0 > kLongRow) continue;
            double bs = 0.0;
            int bi = -1;
            row_hopmax(A, g.ms, g.mi, j, e0, e1, 1, bs, bi);
            g.owner[j] = (bi >= 0 && !(bs < g.sc[j])) ? bi : -1;
        }
        agg_long(
            g, nlong, team, lane, w, nw, [&](int j) { return g.st[j] == 0; }, hopmax,
            [&](int j, double bs, int bi) { g.owner[j] = (bi >= 0 && !(bs < g.sc[j])) ? bi : -1; });
        grid.sync();
        AGG_STAMP(5);
        // admission fixpoint (uncapped sweeps of K/numba_backend.py:235-273)
        // Plain (L1-cacheable) reads: a read may miss an admission made in
        // the same sweep, which only defers it to the next sweep -- the
        // fixpoint (and so the result) is the same; grid.sync() between
        // sweeps makes every earlier admission visible.
        uint8_t* adm = g.adm;
        const bool sym = g.symc[0] == 0 && g.symc[1] == g.symc[2];  // shortcut valid
        while (true) {
            const int slot = itg % 3;
            if (tid == 0) ctl[6 + (itg + 1) % 3] = 0;
            int ch = 0;
            for (int t = tid; t < U.cnt; t += nth) {
                const int j = U[t];
                const int c = g.owner[j];
                const int e0 = A.rp[j], e1 = A.rp[j + 1];
                if (c < 0 || c == j || adm[j] || e1 - e0 > kLongRow) continue;
                bool f = false;
                for (int eb = e0; eb < e1 && !f; eb += 8) {
                    int nb[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) nb[q] = eb + q < e1 ? __ldg(A.ci + eb + q) : j;  // j: not admitted
                    uint8_t av[8];
                    int ov[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) { av[q] = adm[nb[q]]; ov[q] = g.owner[nb[q]]; }
#pragma unroll
                    for (int q = 0; q < 8; ++q) f |= av[q] && ov[q] == c;
                    // j is admitted: so is every same-owner neighbour already
                    // loaded (the fixpoint is reachability from the center
                    // through same-owner vertices, so admitting them now only
                    // shortens the sweep chain; owner == a current center
                    // implies the vertex is in U)
                    if (f && sym) {
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            if (!av[q] && ov[q] == c && nb[q] != c && nb[q] != j) adm[nb[q]] = 1;
                    }
                }
                if (f) { adm[j] = 1; ch = 1; }
            }
            agg_long(
                g, nlong, team, lane, w, nw,
                [&](int j) {  // in U, claimed by another center, not yet admitted
                    const int c = g.owner[j];
                    return g.st[j] != 2 && c >= 0 && c != j && !adm[j];
                },
                [&](int j, int e, int e1, int step, double& bs, int& bi) {
                    const int c = g.owner[j];
                    bool f = false;
                    for (; e < e1 && !f; e += 4 * step) {
                        int nb[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) nb[q] = e + step * q < e1 ? __ldg(A.ci + e + step * q) : j;
                        uint8_t av[4];
                        int ov[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) { av[q] = adm[nb[q]]; ov[q] = g.owner[nb[q]]; }
#pragma unroll
                        for (int q = 0; q < 4; ++q) f |= av[q] && ov[q] == c;
                    }
                    if (f) { bs = 0.0; bi = 0; }  // found: any key
                },
                [&](int j, double, int bi) {
                    if (bi >= 0) { adm[j] = 1; ch = 1; }
                });
            if (__any_sync(0xffffffffu, ch) && lane == 0) atomicOr((int*)&ctl[6 + slot], 1);
            grid.sync();
            AGG_STAMP(6);
            const int any = ctl[6 + slot];
            ++itg;
            if (!any) break;
        }
        // commit: admitted vertices and centers are processed, seeded by
        // owner; the rest of U is appended to the next pass's U in the same
        // sweep (block-tiled, so pass 0 keeps vertex order within a tile)
        int* ucnt = (int*)&ctl[11 + ps];
        wl_compact_blk(
            U.cnt,
            [&](int t, int& v) {
                const int j = U[t];
                v = j;
                const uint8_t sj = g.st[j];
                if (sj == 1 || (sj == 0 && adm[j])) {
                    g.seed_of[j] = g.owner[j];
                    g.st[j] = 2;
                    return false;
                }
                return sj == 0;
            },
            unext, ucnt);
        grid.sync();
        AGG_STAMP(7);
        if (g.prof && tid == 0 && pass < 32) {
            g.prof[4 * pass + 2] = H.cnt;
            g.prof[4 * pass + 3] = itg - itg0;
        }
        remaining = ctl[11 + ps];
        U = WL{unext, remaining};
        if (ctl[ps] == 0) { ++pass; break; }  // no centers (cannot happen, U/aggregation.py:190)
    }
    if (tid == 0) { ctl[9] = pass; ctl[10] = remaining; }
    if (g.prof && tid == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        g.prof[4 * min(pass, 32)] = t;
    }
}

__global__ void __launch_bounds__(256) k_aggregate_coop(AggCoop g) { k_aggregate_body<GridBar>(g); }
__global__ void __launch_bounds__(256) k_aggregate_coop_cg(AggCoop g) { k_aggregate_body<GridBarCg>(g); }
__global__ void __launch_bounds__(kAggClusterThreads, 1) k_aggregate_cluster(AggCoop g) {
    k_aggregate_body<ClusterBar>(g);
}

// ============================================================ renumbering
// leftovers become singletons (U/aggregation.py:195-198); seed flags
__global__ void k_finish_seeds(int n, const uint8_t* st, int* seed_of, int* flag) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        if (st[v] != 2) seed_of[v] = v;
        flag[v] = (seed_of[v] == v);
    }
}
// new id = rank of the seed among all seeds (U/aggregation.py:199-203)
__global__ void k_renumber(int n, const int* seed_of, const int* flag, const int* rank, int* v2a, int* seeds) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        if (flag[v]) seeds[rank[v]] = v;
        v2a[v] = rank[seed_of[v]];
    }
}

// ============================================================ members_csr
__global__ void k_iota(int n, int* v) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) v[i] = i;
}
__global__ void k_seg_starts(int n, int nc, const int* sorted_keys, int* ptr) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int k = sorted_keys[i];
        if (i == 0 || sorted_keys[i - 1] != k) ptr[k] = i;
        if (i == n - 1) ptr[nc] = n;
    }
}

// ============================================================ Galerkin
// stream length per aggregate: sum of its members' row lengths
// stream length of aggregate I = sum of its members' row lengths, row-parallel
// (a thread walking a hub aggregate's thousands of members was 0.4 ms);
// lanes of a warp adding to the same aggregate are merged into one atomic
__global__ void k_stream_len(Csr A, const int* __restrict__ v2a, int* slen) {
    const int lane = threadIdx.x & 31;
    for (int r0 = blockIdx.x * blockDim.x + threadIdx.x - lane; r0 < A.n; r0 += gridDim.x * blockDim.x) {
        const int r = r0 + lane;
        const int I = r < A.n ? v2a[r] : -1;
        const int len = r < A.n ? A.rp[r + 1] - A.rp[r] : 0;
        const unsigned g = __match_any_sync(0xffffffffu, I);
        int tot = 0;
        for (unsigned mm = g; mm; mm &= mm - 1) tot += __shfl_sync(g, len, __ffs(mm) - 1);
        if (I >= 0 && (__ffs(g) - 1) == lane) atomicAdd(slen + I, tot);
    }
}

__device__ __forceinline__ unsigned hslot(int key, int cap) { return ((unsigned)key * 2654435761u) % (unsigned)cap; }
// table capacity of aggregate I's coarse row: at most min(stream length, nc)
// distinct coarse columns, load factor <= 1/2 (fits the 2*slen region at 2*soff)
__device__ __forceinline__ int gal_cap(int L, int nc) { return 2 * min(L, nc); }

// Phase A: one warp per aggregate I accumulates its coarse row in an
// open-addressing table at hkey/hval[2*soff[I] .. +2*slen[I]).  The stream
// (members ascending, each row's entries ascending) is consumed 32 entries
// at a time; lanes with equal J are grouped with __match_any_sync and the
// lowest lane adds the group's values in lane order -- so every (I,J) sum is
// sequential in the reference's stable-sort order (K/numba_backend.py:151-163).
__global__ void k_galerkin_accum(Csr A, const int* __restrict__ v2a, int nc, const int* __restrict__ agg_ptr,
                                 const int* __restrict__ members, const int* __restrict__ soff,
                                 const int* __restrict__ slen, int* hkey, double* hval, int* cnt) {
    __shared__ double wvals[8][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int I = blockIdx.x * 8 + wib;
    if (I >= nc) return;
    const int cap = gal_cap(slen[I], nc);
    int* K = hkey + 2 * (size_t)soff[I];
    double* V = hval + 2 * (size_t)soff[I];
    for (int q = agg_ptr[I]; q < agg_ptr[I + 1]; ++q) {
        const int m = members[q];
        const int e0 = A.rp[m], e1 = A.rp[m + 1];
        for (int c0 = e0; c0 < e1; c0 += 32) {
            const int e = c0 + lane;
            const bool act = e < e1;
            const unsigned am = __ballot_sync(0xffffffffu, act);
            int J = -1;
            double a = 0.0;
            if (act) {
                J = __ldg(v2a + __ldg(A.ci + e));
                a = __ldg(A.av + e);
            }
            wvals[wib][lane] = a;
            __syncwarp();
            if (act) {
                const unsigned g = __match_any_sync(am, J);
                if ((__ffs(g) - 1) == lane) {
                    unsigned slot = hslot(J, cap);
                    while (true) {
                        const int prev = atomicCAS(K + slot, -1, J);
                        if (prev == -1 || prev == J) break;
                        slot = (slot + 1 == (unsigned)cap) ? 0u : slot + 1;
                    }
                    volatile double* vs = V + slot;
                    double acc = *vs;
                    unsigned mm = g;
                    while (mm) {
                        const int l = __ffs(mm) - 1;
                        acc = __dadd_rn(acc, wvals[wib][l]);
                        mm &= mm - 1;
                    }
                    *vs = acc;
                }
            }
            __syncwarp();
        }
    }
    __syncwarp();
    // count nonzero sums (exact zeros dropped, K/numba_backend.py:164)
    int c = 0;
    for (int t = lane; t < cap; t += 32)
        if (K[t] >= 0 && V[t] != 0.0) ++c;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) cnt[I] = c;
}

// Order-free Galerkin accumulation, valid when every value of A is an
// integer and nnz * max|a| < 2^52: then every partial sum of every (I,J) entry
// is an exactly representable integer, so any summation order (here: parallel
// atomics) gives the bit-identical result of the reference's sequential sum.
__device__ __forceinline__ void gal_insert_add(int* K, double* V, int cap, int J, double a) {
    unsigned slot = hslot(J, cap);
    while (true) {
        const int prev = atomicCAS(K + slot, -1, J);
        if (prev == -1 || prev == J) break;
        slot = (slot + 1 == (unsigned)cap) ? 0u : slot + 1;
    }
    atomicAdd(V + slot, a);
}
// shared-memory variant: int64 sums (fp64 shared atomics are CAS spin loops;
// integer-valued sums below 2^52 are exact either way)
template <class T>
__device__ __forceinline__ void gal_insert_add_s(int* K, T* V, int cap, int J, T a) {
    unsigned slot = hslot(J, cap);
    while (true) {
        const int prev = atomicCAS(K + slot, -1, J);
        if (prev == -1 || prev == J) break;
        slot = (slot + 1 == (unsigned)cap) ? 0u : slot + 1;
    }
    if constexpr (sizeof(T) == 4)
        atomicAdd(V + slot, a);  // native shared-memory add
    else
        atomicAdd(reinterpret_cast<unsigned long long*>(V + slot), (unsigned long long)a);
}
__global__ void __launch_bounds__(256) k_galerkin_accum_int(Csr A, int nc, const int* __restrict__ v2a,
                                                            const int* __restrict__ soff,
                                                            const int* __restrict__ slen, int* hkey, double* hval,
                                                            const int* __restrict__ longs, const int* __restrict__ nlong) {
    // short rows: one lane per row, the warp stepping through its rows'
    // entries together; lanes hitting the same (I, J) in a step are merged
    // (__match_any_sync) and one atomic adds their sum -- hub aggregates
    // otherwise serialise thousands of same-address atomics in L2.  Rows
    // longer than kLongRow: one warp per row, merged the same way.  Exact for
    // integer values in any grouping.
    __shared__ double wv[8][32];
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, w = tid >> 5, nw = nth >> 5;
    auto merged_add = [&](bool act, int I, int J, double a) {
        const unsigned long long key = act ? ((unsigned long long)(unsigned)I << 32 | (unsigned)J) : ~0ull;
        const unsigned g = __match_any_sync(0xffffffffu, key);
        wv[wib][lane] = a;
        __syncwarp();
        if (act && (__ffs(g) - 1) == lane) {
            double sum = 0.0;
            for (unsigned mm = g; mm; mm &= mm - 1) sum += wv[wib][__ffs(mm) - 1];
            gal_insert_add(hkey + 2 * (size_t)soff[I], hval + 2 * (size_t)soff[I], gal_cap(slen[I], nc), J, sum);
        }
        __syncwarp();
    };
    for (int r0 = tid - lane; r0 < A.n; r0 += nth) {
        const int r = r0 + lane;
        int e0 = 0, len = 0, I = 0;
        if (r < A.n) {
            e0 = A.rp[r];
            len = A.rp[r + 1] - e0;
            if (len > kLongRow) len = 0;
            I = v2a[r];
        }
        const int mx = __reduce_max_sync(0xffffffffu, len);
        for (int k = 0; k < mx; ++k) {
            const bool act = k < len;
            const int J = act ? __ldg(v2a + __ldg(A.ci + e0 + k)) : -1;
            const double a = act ? __ldg(A.av + e0 + k) : 0.0;
            merged_add(act, I, J, a);
        }
    }
    // long rows (listed by k_long_rows): chunks of 32 entries spread over
    // all warps -- a hub row of thousands of entries walked by one warp is a
    // serial chain of dependent gathers and atomics
    const int nl = *nlong;
    for (int li = 0; li < nl; ++li) {
        const int r = longs[li];
        const int e0 = A.rp[r], e1 = A.rp[r + 1];
        const int I = v2a[r];
        const int nch = (e1 - e0 + 31) >> 5;
        // rotate the starting warp per row so short lists still spread
        for (int c = (w + li * 7) % nw; c < nch; c += nw) {
            const int e = e0 + (c << 5) + lane;
            const bool act = e < e1;
            merged_add(act, I, act ? __ldg(v2a + __ldg(A.ci + e)) : -1, act ? __ldg(A.av + e) : 0.0);
        }
    }
}
// Integer path on levels whose aggregate streams are all short (fine
// levels), one warp per aggregate I: its coarse row accumulated in a
// warp-private open-addressing table in shared memory, the member rows'
// entries flattened across the lanes 32 at a time (a shuffle scan of the
// member row lengths + a shuffle binary search per entry), then the nonzero
// entries compacted, unsorted, into tk/tv at soff[I] and their count into
// cnt[I].  Exact for integer values (any order), like the global tables of
// k_galerkin_accum_int, without scattered DRAM atomics.
constexpr int kGalWarps = 8;
constexpr int kGalStreamMax = 256;          // levels whose longest stream is longer take the global tables
constexpr int kGalCap = 2 * kGalStreamMax;  // shared-memory table slots per warp (load <= 1/2)
template <class T>  // int when every stream's |sum| < 2^31 (native atomics), else long long
__global__ void __launch_bounds__(32 * kGalWarps) k_galerkin_int_warp(Csr A, int nc, const int* __restrict__ v2a,
                                                                     const int* __restrict__ agg_ptr,
                                                                     const int* __restrict__ members,
                                                                     const int* __restrict__ soff,
                                                                     const int* __restrict__ slen, int* tk,
                                                                     double* tv, int* cnt) {
    __shared__ int sk[kGalWarps][kGalCap];
    __shared__ T sv[kGalWarps][kGalCap];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    for (int I = blockIdx.x * kGalWarps + wib; I < nc; I += gridDim.x * kGalWarps) {
        const int L = slen[I];
        const int need = gal_cap(L, nc);
        int cap = 32;
        while (cap < need) cap <<= 1;  // <= kGalCap on this path (every stream <= kGalStreamMax)
        int* K = sk[wib];
        T* V = sv[wib];
        for (int t = lane; t < cap; t += 32) {
            K[t] = -1;
            V[t] = 0;
        }
        __syncwarp();
        const int m0 = agg_ptr[I], m1 = agg_ptr[I + 1];
        for (int mb = m0; mb < m1; mb += 32) {
            const int m = mb + lane < m1 ? members[mb + lane] : -1;
            const int rb = m >= 0 ? A.rp[m] : 0;
            const int len = m >= 0 ? A.rp[m + 1] - rb : 0;
            int pre = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, pre, o);
                if (lane >= o) pre += y;
            }
            const int total = __shfl_sync(0xffffffffu, pre, 31);
            const int excl = pre - len;
            for (int base = 0; base < total; base += 32) {
                const int sidx = base + lane;
                int j = 0;
#pragma unroll
                for (int step = 16; step > 0; step >>= 1) {
                    const int c = j + step;
                    const int ex = __shfl_sync(0xffffffffu, excl, c & 31);
                    if (c < 32 && ex <= sidx) j = c;
                }
                const int rbj = __shfl_sync(0xffffffffu, rb, j);
                const int exj = __shfl_sync(0xffffffffu, excl, j);
                if (sidx < total) {
                    const int e = rbj + (sidx - exj);
                    gal_insert_add_s(K, V, cap, __ldg(v2a + __ldg(A.ci + e)), (T)__ldg(A.av + e));
                }
            }
        }
        __syncwarp();
        // drop exact zeros (K/numba_backend.py:164) compacting the kept
        // entries in place to the front of the table, then write each at its
        // rank among the row's keys: the row leaves here sorted by coarse
        // column, so no segmented sort is needed afterwards
        int c = 0;
        for (int t0 = 0; t0 < cap; t0 += 32) {
            const int t = t0 + lane;
            int key = -1;
            T v = 0;
            if (t < cap) {
                key = K[t];
                v = V[t];
            }
            const bool keep = key >= 0 && v != 0;
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            __syncwarp();  // the round's reads precede its writes (positions <= t)
            if (keep) {
                const int pos = c + __popc(bal & ((1u << lane) - 1u));
                K[pos] = key;
                V[pos] = v;
            }
            c += __popc(bal);
            __syncwarp();
        }
        const size_t o = (size_t)soff[I];
        for (int t = lane; t < c; t += 32) {
            const int key = K[t];
            int rank = 0;
            for (int u = 0; u < c; ++u) rank += K[u] < key;  // broadcast reads
            tk[o + rank] = key;
            tv[o + rank] = (double)V[t];
        }
        if (lane == 0) cnt[I] = c;
        __syncwarp();
    }
}
// move each row's compacted entries to its CSR position
__global__ void k_galerkin_place(int nc, const int* __restrict__ soff, const int* __restrict__ cnt,
                                 const int* __restrict__ rp_c, const int* __restrict__ tk,
                                 const double* __restrict__ tv, int* col_c, double* val_c) {
    const int lane = threadIdx.x & 31;
    for (int I = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; I < nc; I += (gridDim.x * blockDim.x) >> 5) {
        const size_t o = (size_t)soff[I];
        const int b = rp_c[I];
        for (int t = lane; t < cnt[I]; t += 32) {
            col_c[b + t] = tk[o + t];
            val_c[b + t] = tv[o + t];
        }
    }
}
__global__ void k_galerkin_count(int nc, const int* __restrict__ soff, const int* __restrict__ slen,
                                 const int* __restrict__ hkey, const double* __restrict__ hval, int* cnt) {
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int I = blockIdx.x * 8 + wib;
    if (I >= nc) return;
    const int cap = gal_cap(slen[I], nc);
    const int* K = hkey + 2 * (size_t)soff[I];
    const double* V = hval + 2 * (size_t)soff[I];
    int c = 0;
    for (int t = lane; t < cap; t += 32) c += (K[t] >= 0 && V[t] != 0.0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) cnt[I] = c;
}
// integrality test for the order-free path
__global__ void k_int_check(long long m, const double* __restrict__ v, int* nonint, unsigned long long* maxabs) {
    double mx = 0.0;
    int bad = 0;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < m; k += (long long)gridDim.x * blockDim.x) {
        const double a = v[k];
        bad |= (a != rint(a));
        mx = fmax(mx, fabs(a));
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonint, 1);
    mx = block_max(mx);
    if (threadIdx.x == 0) atomicMax(maxabs, (unsigned long long)__double_as_longlong(mx));
}

// Phase C: compact the nonzero (J, value) pairs of row I to its output slot
// range (slot order); rows are then sorted by J with a segmented sort.
__global__ void k_galerkin_compact(int nc, const int* __restrict__ soff, const int* __restrict__ slen,
                                   const int* __restrict__ hkey, const double* __restrict__ hval,
                                   const int* __restrict__ rp_c, int* col_c, double* val_c) {
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int I = blockIdx.x * 8 + wib;
    if (I >= nc) return;
    const int cap = gal_cap(slen[I], nc);
    const int* K = hkey + 2 * (size_t)soff[I];
    const double* V = hval + 2 * (size_t)soff[I];
    int base = rp_c[I];
    for (int t0 = 0; t0 < cap; t0 += 32) {
        const int t = t0 + lane;
        int key = -1;
        double v = 0.0;
        if (t < cap) { key = K[t]; v = V[t]; }
        const bool keep = key >= 0 && v != 0.0;
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (keep) {
            const int pos = base + __popc(m & ((1u << lane) - 1u));
            col_c[pos] = key;
            val_c[pos] = v;
        }
        base += __popc(m);
    }
}

// ============================================================ coarsest dense
__global__ void k_densify(Csr A, double* D) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += gridDim.x * blockDim.x)
        for (int k = A.rp[i]; k < A.rp[i + 1]; ++k) D[(size_t)i * A.n + A.ci[k]] = A.av[k];
}

// in-place lower Cholesky (row-major, lower triangle), single block; flag on
// a non-positive pivot (scipy cho_factor LinAlgError, U/hierarchy.py:47-51)
__global__ void k_cholesky(int n, double* L, int* fail) {
    __shared__ double piv;
    for (int j = 0; j < n; ++j) {
        if (threadIdx.x == 0) {
            double s = L[(size_t)j * n + j];
            for (int k = 0; k < j; ++k) s -= L[(size_t)j * n + k] * L[(size_t)j * n + k];
            if (!(s > 0.0)) { *fail = 1; piv = 0.0; }
            else { piv = sqrt(s); L[(size_t)j * n + j] = piv; }
        }
        __syncthreads();
        if (piv == 0.0) return;
        for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) {
            double s = L[(size_t)i * n + j];
            for (int k = 0; k < j; ++k) s -= L[(size_t)i * n + k] * L[(size_t)j * n + k];
            L[(size_t)i * n + j] = s / piv;
        }
        __syncthreads();
    }
}
// inverse from the Cholesky factor: column c of A^{-1} per thread
__global__ void k_chol_inverse(int n, const double* L, double* Minv, double* work) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n) return;
    double* y = work + (size_t)c * n;
    for (int i = 0; i < n; ++i) {  // L y = e_c
        double s = (i == c) ? 1.0 : 0.0;
        for (int k = 0; k < i; ++k) s -= L[(size_t)i * n + k] * y[k];
        y[i] = s / L[(size_t)i * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {  // L^T x = y
        double s = y[i];
        for (int k = i + 1; k < n; ++k) s -= L[(size_t)k * n + i] * y[k];
        y[i] = s / L[(size_t)i * n + i];
    }
    for (int i = 0; i < n; ++i) Minv[(size_t)i * n + c] = y[i];
}

// cyclic Jacobi eigen-decomposition (single block) for the singular /
// indefinite fallback (numpy eigh, U/hierarchy.py:52-54)
__global__ void k_jacobi_eigh(int n, double* A, double* V, int sweeps) {
    __shared__ double cs, sn;
    __shared__ int skip;
    for (int t = threadIdx.x; t < n * n; t += blockDim.x) V[t] = ((t / n) == (t % n)) ? 1.0 : 0.0;
    __syncthreads();
    __shared__ double red[256];
    for (int sw = 0; sw < sweeps; ++sw) {
        // stop when the off-diagonal mass is negligible
        double off = 0.0, tot = 0.0;
        for (int t = threadIdx.x; t < n * n; t += blockDim.x) {
            const double v = A[t] * A[t];
            tot += v;
            if ((t / n) != (t % n)) off += v;
        }
        red[threadIdx.x] = off;
        __syncthreads();
        if (threadIdx.x == 0) {
            double o = 0.0;
            for (int k = 0; k < (int)blockDim.x; ++k) o += red[k];
            red[0] = o;
        }
        __syncthreads();
        const double offs = red[0];
        __syncthreads();
        red[threadIdx.x] = tot;
        __syncthreads();
        if (threadIdx.x == 0) {
            double o = 0.0;
            for (int k = 0; k < (int)blockDim.x; ++k) o += red[k];
            red[0] = o;
        }
        __syncthreads();
        const double tots = red[0];
        __syncthreads();
        if (offs <= 1e-30 * (tots > 0.0 ? tots : 1.0)) break;
        for (int p = 0; p < n; ++p) {
            for (int q = p + 1; q < n; ++q) {
                if (threadIdx.x == 0) {
                    const double apq = A[(size_t)p * n + q];
                    skip = fabs(apq) < 1e-300;
                    if (!skip) {
                        const double app = A[(size_t)p * n + p], aqq = A[(size_t)q * n + q];
                        const double th = (aqq - app) / (2.0 * apq);
                        const double t = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
                        cs = 1.0 / sqrt(t * t + 1.0);
                        sn = t * cs;
                    }
                }
                __syncthreads();
                if (!skip) {
                    const double c = cs, s = sn;
                    for (int k = threadIdx.x; k < n; k += blockDim.x) {
                        const double akp = A[(size_t)k * n + p], akq = A[(size_t)k * n + q];
                        A[(size_t)k * n + p] = c * akp - s * akq;
                        A[(size_t)k * n + q] = s * akp + c * akq;
                    }
                    __syncthreads();
                    for (int k = threadIdx.x; k < n; k += blockDim.x) {
                        const double apk = A[(size_t)p * n + k], aqk = A[(size_t)q * n + k];
                        A[(size_t)p * n + k] = c * apk - s * aqk;
                        A[(size_t)q * n + k] = s * apk + c * aqk;
                        const double vkp = V[(size_t)k * n + p], vkq = V[(size_t)k * n + q];
                        V[(size_t)k * n + p] = c * vkp - s * vkq;
                        V[(size_t)k * n + q] = s * vkp + c * vkq;
                    }
                }
                __syncthreads();
            }
        }
    }
}
// pinv = V diag(inv) V^T with cut = 1e-12 * max(lambda_max, 0)
__global__ void k_pinv(int n, const double* A, const double* V, double* M) {
    __shared__ double lmax;
    if (threadIdx.x == 0) {
        double m = -1e300;
        for (int k = 0; k < n; ++k) m = fmax(m, A[(size_t)k * n + k]);
        lmax = m;
    }
    __syncthreads();
    const double cut = 1e-12 * fmax(lmax, 0.0);
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n * n; t += gridDim.x * blockDim.x) {
        const int i = t / n, j = t % n;
        double s = 0.0;
        for (int k = 0; k < n; ++k) {
            const double w = A[(size_t)k * n + k];
            if (w > cut) s += V[(size_t)i * n + k] * (1.0 / w) * V[(size_t)j * n + k];
        }
        M[t] = s;
    }
}

// ============================================================ squared pattern (kernel table)
__global__ void k_sq_count(Csr A, long long* cnt) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += gridDim.x * blockDim.x) {
        long long c = 0;
        for (int e = A.rp[i]; e < A.rp[i + 1]; ++e) {
            const int k = A.ci[e];
            c += A.rp[k + 1] - A.rp[k];
        }
        cnt[i] = c;
    }
}
__global__ void k_sq_expand(Csr A, const long long* off, unsigned long long* keys) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += gridDim.x * blockDim.x) {
        long long p = off[i];
        for (int e = A.rp[i]; e < A.rp[i + 1]; ++e) {
            const int k = A.ci[e];
            for (int e2 = A.rp[k]; e2 < A.rp[k + 1]; ++e2)
                keys[p++] = ((unsigned long long)i << 32) | (unsigned)A.ci[e2];
        }
    }
}

// ============================================================ host drivers
static int grid_for(int n) { return std::max(1, std::min(cdiv(n, 256), 4 * kNumSMs)); }

// Grow-only per-thread scratch for the large transient setup buffers (the
// Galerkin hash, the aggregation state): a setup finishes all its device
// work before returning, so the next setup issued by the same thread can
// reuse the memory; no pool growth or page mapping inside the timed setup.
struct Scratch {
    void* p = nullptr;
    size_t bytes = 0;
    ~Scratch() {
        if (p) cudaFree(p);
    }
};
template <class T>
static T* scratch(int slot, size_t count) {
    static thread_local Scratch slots[kMaxDevices][16];
    Scratch& sl = slots[cur_dev()][slot];
    const size_t want = count * sizeof(T) + 64;
    if (want > sl.bytes) {
        if (sl.p) {
            UA_CK(cudaDeviceSynchronize());
            UA_CK(cudaFree(sl.p));
            sl.p = nullptr;
        }
        const size_t grow = want + want / 4;
        UA_CK(cudaMalloc(&sl.p, grow));
        sl.bytes = grow;
    }
    return static_cast<T*>(sl.p);
}

template <class T>
struct SPtr {
    T* p;
};

template <class T>
static void exclusive_scan(const T* in, T* out, int n, cudaStream_t s) {
    size_t tmp = 0;
    UA_CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, s));
    DBuf<char> t(tmp, s);
    UA_CK(cub::DeviceScan::ExclusiveSum(t.p, tmp, in, out, n, s));
}

// aggregate() on device.  state arrays are n-sized scratch.
int device_aggregate(const Csr& A, const int* deg, uint64_t seed, int max_passes, long long size_cap,
                     int* v2a, int* seeds, cudaStream_t s, AggStats* stats, const std::function<void()>* overlap) {
    const int n = A.n;
    if (n <= 0) throw Error(UAAMG_EAGG, "cannot aggregate an empty matrix");
    if (overlap && size_cap > 0) (*overlap)();
    const int G = grid_for(n);
    SPtr<uint8_t> st{scratch<uint8_t>(2, n)}, adm{scratch<uint8_t>(3, n)};
    SPtr<double> sc{scratch<double>(4, n)}, ms{scratch<double>(5, n)};
    SPtr<int> mi{scratch<int>(6, n)}, owner{scratch<int>(7, n)}, seed_of{scratch<int>(8, n)};
    DBuf<int> counters(4, s);
    UA_CK(cudaMemsetAsync(st.p, 0, n, s));
    UA_CK(cudaMemsetAsync(seed_of.p, 0xff, sizeof(int) * n, s));
    static thread_local int* h_cnt = nullptr;  // pinned, reused across calls
    if (!h_cnt) UA_CK(cudaMallocHost(&h_cnt, 4 * sizeof(int)));
    const bool capped = size_cap > 0;
    DBuf<int> bcnt, bptr, bjs, ord, cursor;
    DBuf<double> bw;
    DBuf<uint8_t> badm, newly;
    if (capped) {
        bcnt.alloc(n + 1, s); bptr.alloc(n + 1, s); bjs.alloc(n, s); ord.alloc(n, s); cursor.alloc(n, s);
        bw.alloc(n, s); badm.alloc(n, s); newly.alloc(n, s);
        UA_CK(cudaMemsetAsync(newly.p, 0, n, s));
    }
    int passes = 0;
    int remaining = n;
    if (!capped) {
        DBuf<int> ctl(24, s);
        SPtr<int> ul0{scratch<int>(9, n)}, ul1{scratch<int>(10, n)}, hl{scratch<int>(11, n)}, mark{scratch<int>(12, n)};
        UA_CK(cudaMemsetAsync(ctl.p, 0, 24 * sizeof(int), s));
        UA_CK(cudaMemsetAsync(mark.p, 0, sizeof(int) * n, s));
        SPtr<int> longs{scratch<int>(13, n)};
        UA_LAUNCH(k_long_rows, std::min(cdiv(n, 256), 4 * 148), 256, 0, s, A, longs.p, ctl.p + 16);
        DBuf<int> symc(3, s);
        UA_CK(cudaMemsetAsync(symc.p, 0, 3 * sizeof(int), s));
        UA_LAUNCH(k_pattern_sym, std::min(cdiv((long long)n * 32, 256), 16 * 148), 256, 0, s, A, symc.p);
        AggCoop g;
        g.symc = symc.p;
        g.A = A;
        g.longs = longs.p;
        g.nlongs = ctl.p + 16; g.deg = deg; g.seed = seed; g.max_passes = max_passes; g.st = st.p; g.sc = sc.p; g.ms = ms.p;
        g.mi = mi.p; g.owner = owner.p; g.adm = adm.p; g.seed_of = seed_of.p; g.ctl = ctl.p;
        g.ulist[0] = ul0.p; g.ulist[1] = ul1.p; g.hlist = hl.p; g.mark = mark.p;
        static const bool aprof = getenv("UAAMG_AGG_PROF") != nullptr;
        DBuf<unsigned long long> prof;
        g.prof = nullptr;
        if (aprof) {
            prof.alloc(4 * 33 + 40, s);
            UA_CK(cudaMemsetAsync(prof.p, 0, sizeof(unsigned long long) * (4 * 33 + 40), s));
            g.prof = prof.p;
        }
        static int max_blocks_dev[kMaxDevices] = {};
        int& max_blocks = max_blocks_dev[cur_dev()];
        if (!max_blocks) {
            int per_sm = 0, dev = 0, sms = 0;
            UA_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_aggregate_coop, 256, 0));
            UA_CK(cudaGetDevice(&dev));
            UA_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
            max_blocks = std::max(1, per_sm) * sms;
        }
        // one vertex per thread up to full residency: the passes are
        // latency-bound, fewer CTAs (cheaper barriers) measured slower
        int blocks = std::max(1, std::min(max_blocks, cdiv(n, 256)));
        static const bool no_cluster = getenv("UAAMG_AGG_NO_CLUSTER") != nullptr;  // A/B diagnostics
        static const int cl_max = getenv("UAAMG_AGG_CLUSTER_MAX") ? atoi(getenv("UAAMG_AGG_CLUSTER_MAX"))
                                                                  : kAggClusterMaxRows;  // A/B diagnostics
        if (n <= cl_max && !no_cluster) {
            // small level: every pass is a chain of latency-bound phases;
            // one 16-CTA cluster with hardware barriers instead of the grid
            static bool attr_dev[kMaxDevices] = {};
            bool& attr = attr_dev[cur_dev()];
            if (!attr) {
                UA_CK(cudaFuncSetAttribute(k_aggregate_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
                attr = true;
            }
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(kAggClusterCtas);
            cfg.blockDim = dim3(kAggClusterThreads);
            cfg.stream = s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = kAggClusterCtas;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            UA_CK(cudaLaunchKernelEx(&cfg, k_aggregate_cluster, g));
            blocks = kAggClusterCtas;
        } else {
            void* args[] = {&g};
            static const bool cg_sync = getenv("UAAMG_AGG_CG_SYNC") != nullptr;  // A/B diagnostics
            UA_CK(cudaLaunchCooperativeKernel(cg_sync ? (void*)k_aggregate_coop_cg : (void*)k_aggregate_coop, blocks,
                                              256, args, 0, s));
        }
        g_launches.fetch_add(1, std::memory_order_relaxed);
        if (overlap) (*overlap)();
        UA_CK(cudaMemcpyAsync(h_cnt, ctl.p + 9, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
        UA_CK(cudaStreamSynchronize(s));
        passes = h_cnt[0];
        remaining = h_cnt[1];
        max_passes = 0;  // skip the host-driven loop below
        if (aprof) {
            unsigned long long hp[4 * 33 + 40];
            UA_CK(cudaMemcpy(hp, prof.p, sizeof(hp), cudaMemcpyDeviceToHost));
            for (int ps = 0; ps < 2; ++ps) {
                fprintf(stderr, "  pass %d phases (us):", ps);
                unsigned long long prev = hp[4 * ps];
                for (int q = 0; q < 16; ++q) {
                    const unsigned long long v = hp[140 + ps * 16 + q];
                    if (!v) continue;
                    fprintf(stderr, " %d:%.1f", q, (v - prev) * 1e-3);
                    prev = v;
                }
                fprintf(stderr, "\n");
            }
            fprintf(stderr, "aggregate n=%d blocks=%d passes=%d\n", n, blocks, passes);
            for (int k = 0; k < std::min(passes, 32); ++k)
                fprintf(stderr, "  pass %2d |U| %9llu |H| %9llu adm-it %2llu  %8.1f us\n", k, hp[4 * k + 1],
                        hp[4 * k + 2], hp[4 * k + 3], (hp[4 * (k + 1)] - hp[4 * k]) * 1e-3);
        }
    }
    for (int pass = 0; pass < max_passes; ++pass) {
        if (remaining == 0) break;  // U/aggregation.py:186
        UA_CK(cudaMemsetAsync(counters.p, 0, 4 * sizeof(int), s));
        launch_scores(A, deg, seed, pass, sc.p, s);
        UA_LAUNCH(k_hop1, G, 256, 0, s, A, sc.p, st.p, 0, ms.p, mi.p);
        UA_LAUNCH(k_select, G, 256, 0, s, A, sc.p, st.p, ms.p, mi.p, counters.p + 0);
        UA_LAUNCH(k_hop1, G, 256, 0, s, A, sc.p, st.p, 1, ms.p, mi.p);
        UA_LAUNCH(k_claim, G, 256, 0, s, A, sc.p, st.p, ms.p, mi.p, owner.p);
        if (!capped) {
            UA_LAUNCH(k_admit_init, G, 256, 0, s, n, st.p, owner.p, adm.p);
            for (int it = 0; it < n + 1; ++it) {
                UA_CK(cudaMemsetAsync(counters.p + 1, 0, sizeof(int), s));
                UA_LAUNCH(k_admit_step, G, 256, 0, s, A, owner.p, adm.p, counters.p + 1);
                UA_CK(cudaMemcpyAsync(h_cnt + 1, counters.p + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
                UA_CK(cudaStreamSynchronize(s));
                if (h_cnt[1] == 0) break;
            }
            UA_LAUNCH(k_admit_commit, G, 256, 0, s, n, st.p, owner.p, adm.p, seed_of.p, counters.p + 2);
        } else {
            UA_CK(cudaMemsetAsync(bcnt.p, 0, sizeof(int) * (n + 1), s));
            UA_CK(cudaMemsetAsync(cursor.p, 0, sizeof(int) * n, s));
            UA_LAUNCH(k_bucket_count, G, 256, 0, s, n, st.p, owner.p, bcnt.p);
            exclusive_scan(bcnt.p, bptr.p, n + 1, s);
            UA_LAUNCH(k_bucket_fill, G, 256, 0, s, n, st.p, owner.p, bptr.p, cursor.p, bjs.p);
            UA_LAUNCH(k_admit_capped, G, 256, 0, s, A, n, st.p, bptr.p, bjs.p, ord.p, bw.p, badm.p, size_cap,
                      seed_of.p, newly.p);
            UA_LAUNCH(k_capped_commit, G, 256, 0, s, n, st.p, newly.p, counters.p + 2);
        }
        UA_CK(cudaMemcpyAsync(h_cnt, counters.p, 4 * sizeof(int), cudaMemcpyDeviceToHost, s));
        UA_CK(cudaStreamSynchronize(s));
        ++passes;
        remaining = h_cnt[2];
        if (h_cnt[0] == 0) break;  // no centers: cannot happen (U/aggregation.py:190)
    }
    // leftovers + renumber
    DBuf<int> flag(n + 1, s), rank(n + 1, s);
    UA_LAUNCH(k_finish_seeds, G, 256, 0, s, n, st.p, seed_of.p, flag.p);
    UA_CK(cudaMemsetAsync(flag.p + n, 0, sizeof(int), s));
    exclusive_scan(flag.p, rank.p, n + 1, s);
    UA_LAUNCH(k_renumber, G, 256, 0, s, n, seed_of.p, flag.p, rank.p, v2a, seeds);
    int nc = 0;
    UA_CK(cudaMemcpyAsync(&nc, rank.p + n, sizeof(int), cudaMemcpyDeviceToHost, s));
    UA_CK(cudaStreamSynchronize(s));
    if (stats) { stats->passes = passes; stats->leftover = remaining; }
    return nc;
}

void build_members(int n, int nc, const int* v2a, int* agg_ptr, int* members, cudaStream_t s) {
    DBuf<int> iota(n, s), keys_out(n, s);
    UA_LAUNCH(k_iota, grid_for(n), 256, 0, s, n, iota.p);
    int bits = 1;
    while ((1ll << bits) < (long long)nc) ++bits;
    size_t tmp = 0;
    UA_CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, v2a, keys_out.p, iota.p, members, n, 0, bits, s));
    DBuf<char> t(tmp, s);
    UA_CK(cub::DeviceRadixSort::SortPairs(t.p, tmp, v2a, keys_out.p, iota.p, members, n, 0, bits, s));
    UA_LAUNCH(k_seg_starts, grid_for(n), 256, 0, s, n, nc, keys_out.p, agg_ptr);
}


// Galerkin: returns nnz_c; allocates out arrays
long long device_galerkin(const Csr& A, const int* v2a, int nc, const int* agg_ptr, const int* members,
                          DBuf<int>& rp_c, DBuf<int>& ci_c, DBuf<double>& av_c, cudaStream_t s) {
    static const bool gprof = getenv("UAAMG_GAL_PROF") != nullptr;  // diagnostics: per-step stream time
    auto gt = [&](const char* tag) {
        if (!gprof) return;
        static auto last = std::chrono::steady_clock::now();
        UA_CK(cudaStreamSynchronize(s));
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "  galerkin nc=%d %-10s %8.3f ms\n", nc, tag, std::chrono::duration<double, std::milli>(now - last).count());
        last = now;
    };
    gt("start");
    DBuf<int> slen(nc + 1, s), soff(nc + 1, s), cnt(nc + 1, s);
    UA_CK(cudaMemsetAsync(slen.p, 0, sizeof(int) * nc, s));
    UA_LAUNCH(k_stream_len, grid_for(A.n), 256, 0, s, A, v2a, slen.p);
    UA_CK(cudaMemsetAsync(slen.p + nc, 0, sizeof(int), s));
    exclusive_scan(slen.p, soff.p, nc + 1, s);
    gt("slen");
    const size_t hsz = 2 * (size_t)std::max(A.nnz, 1);
    SPtr<int> hkey{scratch<int>(0, hsz)};
    SPtr<double> hval{scratch<double>(1, hsz)};
    // integrality / magnitude of A and the longest aggregate stream, read
    // back together (one host round trip chooses the path)
    bool exact_int = true, warp_path = false;
    double maxabs = 0.0;
    if (A.nnz > 0) {
        DBuf<int> bad(1, s), smx(1, s);
        DBuf<unsigned long long> amx(1, s);
        UA_CK(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
        UA_CK(cudaMemsetAsync(amx.p, 0, sizeof(unsigned long long), s));
        UA_LAUNCH(k_int_check, grid_for(A.nnz), 256, 0, s, (long long)A.nnz, A.av, bad.p, amx.p);
        size_t tmp = 0;
        UA_CK(cub::DeviceReduce::Max(nullptr, tmp, slen.p, smx.p, nc, s));
        DBuf<char> t(tmp, s);
        UA_CK(cub::DeviceReduce::Max(t.p, tmp, slen.p, smx.p, nc, s));
        int h_bad = 0, h_smx = 0;
        unsigned long long h_amx = 0;
        UA_CK(cudaMemcpyAsync(&h_bad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        UA_CK(cudaMemcpyAsync(&h_amx, amx.p, sizeof(h_amx), cudaMemcpyDeviceToHost, s));
        UA_CK(cudaMemcpyAsync(&h_smx, smx.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        UA_CK(cudaStreamSynchronize(s));
        std::memcpy(&maxabs, &h_amx, 8);
        exact_int = h_bad == 0 && (double)A.nnz * maxabs < 4503599627370496.0;  // 2^52
        // warp-per-aggregate shared-memory tables when every aggregate's
        // stream is short (fine levels); otherwise (hub aggregates of coarse
        // levels) the all-threads global table, whose parallelism does not
        // depend on the longest stream
        warp_path = exact_int && h_smx <= kGalStreamMax;
    }
    gt("intcheck");
    SPtr<int> tk{nullptr};
    SPtr<double> tv{nullptr};
    if (exact_int && !warp_path) {
        UA_CK(cudaMemsetAsync(hkey.p, 0xff, sizeof(int) * hsz, s));
        UA_CK(cudaMemsetAsync(hval.p, 0, sizeof(double) * hsz, s));
        DBuf<int> nlong(1, s);
        SPtr<int> longs{scratch<int>(13, (size_t)std::max(A.n, 1))};
        UA_CK(cudaMemsetAsync(nlong.p, 0, sizeof(int), s));
        UA_LAUNCH(k_long_rows, grid_for(A.n), 256, 0, s, A, longs.p, nlong.p);
        UA_LAUNCH(k_galerkin_accum_int, grid_for(A.n), 256, 0, s, A, nc, v2a, soff.p, slen.p, hkey.p, hval.p,
                  longs.p, nlong.p);
        UA_LAUNCH(k_galerkin_count, cdiv(nc, 8), 256, 0, s, nc, soff.p, slen.p, hkey.p, hval.p, cnt.p);
    } else if (exact_int) {
        tk.p = scratch<int>(14, (size_t)std::max(A.nnz, 1));
        tv.p = scratch<double>(15, (size_t)std::max(A.nnz, 1));
        // every stream is <= kGalStreamMax entries of |a| <= maxabs
        if ((double)kGalStreamMax * maxabs < 2147483647.0)
            UA_LAUNCH(k_galerkin_int_warp<int>, std::min(cdiv(nc, kGalWarps), 148 * 16), 32 * kGalWarps, 0, s, A, nc,
                      v2a, agg_ptr, members, soff.p, slen.p, tk.p, tv.p, cnt.p);
        else
            UA_LAUNCH(k_galerkin_int_warp<long long>, std::min(cdiv(nc, kGalWarps), 148 * 16), 32 * kGalWarps, 0, s, A,
                      nc, v2a, agg_ptr, members, soff.p, slen.p, tk.p, tv.p, cnt.p);

    } else {
        UA_CK(cudaMemsetAsync(hkey.p, 0xff, sizeof(int) * hsz, s));
        UA_CK(cudaMemsetAsync(hval.p, 0, sizeof(double) * hsz, s));
        UA_LAUNCH(k_galerkin_accum, cdiv(nc, 8), 256, 0, s, A, v2a, nc, agg_ptr, members, soff.p, slen.p, hkey.p,
                  hval.p, cnt.p);
    }
    gt("accum");
    UA_CK(cudaMemsetAsync(cnt.p + nc, 0, sizeof(int), s));
    rp_c.alloc(nc + 1, s);
    exclusive_scan(cnt.p, rp_c.p, nc + 1, s);
    int nnz_c = 0;
    UA_CK(cudaMemcpyAsync(&nnz_c, rp_c.p + nc, sizeof(int), cudaMemcpyDeviceToHost, s));
    UA_CK(cudaStreamSynchronize(s));
    gt("scan");
    ci_c.alloc(std::max(nnz_c, 1), s);
    av_c.alloc(std::max(nnz_c, 1), s);
    if (nnz_c > 0) {
        if (warp_path) {
            // rows already sorted by the warp kernel: place them straight
            // into the output CSR
            UA_LAUNCH(k_galerkin_place, std::min(cdiv(nc, 8), 148 * 16), 256, 0, s, nc, soff.p, cnt.p, rp_c.p, tk.p,
                      tv.p, ci_c.p, av_c.p);
        } else {
            DBuf<int> ck(nnz_c, s);
            DBuf<double> cv(nnz_c, s);
            UA_LAUNCH(k_galerkin_compact, cdiv(nc, 8), 256, 0, s, nc, soff.p, slen.p, hkey.p, hval.p, rp_c.p, ck.p,
                      cv.p);
            size_t tmp = 0;
            UA_CK(cub::DeviceSegmentedSort::SortPairs(nullptr, tmp, ck.p, ci_c.p, cv.p, av_c.p, nnz_c, nc, rp_c.p,
                                                      rp_c.p + 1, s));
            DBuf<char> t(tmp, s);
            UA_CK(cub::DeviceSegmentedSort::SortPairs(t.p, tmp, ck.p, ci_c.p, cv.p, av_c.p, nnz_c, nc, rp_c.p,
                                                      rp_c.p + 1, s));
        }
    }
    gt("sort");
    return nnz_c;
}

// coarsest: dense inverse (Cholesky) or eigen pseudo-inverse
int device_coarse_factor(const Csr& A, bool singular, DBuf<double>& Minv, cudaStream_t s) {
    const int n = A.n;
    Minv.alloc((size_t)std::max(n, 1) * std::max(n, 1), s);
    if (n == 0) return 0;
    DBuf<double> D((size_t)n * n, s);
    UA_CK(cudaMemsetAsync(D.p, 0, sizeof(double) * n * n, s));
    UA_LAUNCH(k_densify, grid_for(n), 256, 0, s, A, D.p);
    int mode = 2;
    if (!singular) {
        DBuf<double> L((size_t)n * n, s), work((size_t)n * n, s);
        DBuf<int> fail(1, s);
        UA_CK(cudaMemsetAsync(fail.p, 0, sizeof(int), s));
        UA_CK(cudaMemcpyAsync(L.p, D.p, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, s));
        UA_LAUNCH(k_cholesky, 1, 1024, 0, s, n, L.p, fail.p);
        int h_fail = 0;
        UA_CK(cudaMemcpyAsync(&h_fail, fail.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        UA_CK(cudaStreamSynchronize(s));
        if (!h_fail) {
            UA_LAUNCH(k_chol_inverse, cdiv(n, 128), 128, 0, s, n, L.p, Minv.p, work.p);
            mode = 1;
        }
    }
    if (mode == 2) {
        DBuf<double> V((size_t)n * n, s);
        UA_LAUNCH(k_jacobi_eigh, 1, 256, 0, s, n, D.p, V.p, 60);
        UA_LAUNCH(k_pinv, std::min(cdiv((long long)n * n, 256), 1024), 256, 0, s, n, D.p, V.p, Minv.p);
    }
    UA_CK(cudaStreamSynchronize(s));
    return mode;
}

// explicit pattern selection / claim (kernel table)
void launch_select_pattern(const Csr& P, const double* s_, const uint8_t* processed, uint8_t* out, cudaStream_t s) {
    UA_LAUNCH(k_select_pattern, grid_for(P.n), 256, 0, s, P, s_, processed, out);
}
void launch_claim_pattern(const Csr& P, const double* s_, const uint8_t* processed, const uint8_t* is_center,
                          int* owner, cudaStream_t s) {
    UA_LAUNCH(k_claim_pattern, grid_for(P.n), 256, 0, s, P, s_, processed, is_center, owner);
}

// 2-hop selection/claim for the kernel table: processed/is_center -> state
__global__ void k_state_from(int n, const uint8_t* processed, const uint8_t* is_center, uint8_t* st) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        st[i] = processed[i] ? 2 : ((is_center && is_center[i]) ? 1 : 0);
}
__global__ void k_state_to_center(int n, const uint8_t* st, uint8_t* out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = st[i] == 1;
}
void select_2hop(const Csr& A, const double* sc, const uint8_t* processed, uint8_t* out, cudaStream_t s) {
    const int n = A.n, G = grid_for(n);
    DBuf<uint8_t> st(n, s);
    DBuf<double> ms(n, s);
    DBuf<int> mi(n, s), cnt(1, s);
    UA_CK(cudaMemsetAsync(cnt.p, 0, sizeof(int), s));
    UA_LAUNCH(k_state_from, G, 256, 0, s, n, processed, (const uint8_t*)nullptr, st.p);
    UA_LAUNCH(k_hop1, G, 256, 0, s, A, sc, st.p, 0, ms.p, mi.p);
    UA_LAUNCH(k_select, G, 256, 0, s, A, sc, st.p, ms.p, mi.p, cnt.p);
    UA_LAUNCH(k_state_to_center, G, 256, 0, s, n, st.p, out);
}
void claim_2hop(const Csr& A, const double* sc, const uint8_t* processed, const uint8_t* is_center, int* owner,
                cudaStream_t s) {
    const int n = A.n, G = grid_for(n);
    DBuf<uint8_t> st(n, s);
    DBuf<double> ms(n, s);
    DBuf<int> mi(n, s);
    UA_LAUNCH(k_state_from, G, 256, 0, s, n, processed, is_center, st.p);
    UA_LAUNCH(k_hop1, G, 256, 0, s, A, sc, st.p, 1, ms.p, mi.p);
    UA_LAUNCH(k_claim, G, 256, 0, s, A, sc, st.p, ms.p, mi.p, owner);
}

// admit_members with caller-built buckets (kernel table): sequential greedy
// per center, reusing k_admit_capped's logic through a bucket-per-center view
__global__ void k_admit_table(Csr A, int nctr, const int* centers, const int* bptr, const int* bjs, long long cap,
                              uint8_t* processed, int* v2a, int agg_base, int* ord, double* w, uint8_t* admf) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nctr; b += gridDim.x * blockDim.x) {
        const int c = centers[b];
        const int agg = agg_base + b;
        v2a[c] = agg;
        processed[c] = 1;
        const int lo = bptr[b], m = bptr[b + 1] - lo;
        const int* js = bjs + lo;
        int* od = ord + lo;
        double* wv = w + lo;
        uint8_t* ad = admf + lo;
        const int rs = A.rp[c], re = A.rp[c + 1];
        for (int t = 0; t < m; ++t) {
            const int pos = lower_bound_i(A.ci, rs, re, js[t]);
            wv[t] = (pos < re && A.ci[pos] == js[t]) ? fabs(A.av[pos]) : 0.0;
            ad[t] = 0;
            int q = t - 1;
            while (q >= 0 && wv[od[q]] < wv[t]) { od[q + 1] = od[q]; --q; }
            od[q + 1] = t;
        }
        long long count = 1;
        bool progress = true;
        while (progress && count < cap) {
            progress = false;
            for (int t = 0; t < m; ++t) {
                if (count >= cap) break;
                const int id = od[t];
                if (ad[id]) continue;
                const int j = js[id];
                bool conn = false;
                for (int e = A.rp[j]; e < A.rp[j + 1]; ++e) {
                    const int nb = A.ci[e];
                    if (nb == c) { conn = true; break; }
                    const int pos = lower_bound_i(js, 0, m, nb);
                    if (pos < m && js[pos] == nb && ad[pos]) { conn = true; break; }
                }
                if (conn) {
                    ad[id] = 1;
                    v2a[j] = agg;
                    processed[j] = 1;
                    ++count;
                    progress = true;
                }
            }
        }
    }
}
void admit_table(const Csr& A, int nctr, const int* centers, const int* bptr, const int* bjs, long long cap,
                 uint8_t* processed, int* v2a, int agg_base, int total_bucket, cudaStream_t s) {
    const int m = std::max(total_bucket, 1);
    DBuf<int> ord(m, s);
    DBuf<double> w(m, s);
    DBuf<uint8_t> adm(m, s);
    UA_LAUNCH(k_admit_table, grid_for(nctr), 256, 0, s, A, nctr, centers, bptr, bjs, cap, processed, v2a, agg_base,
              ord.p, w.p, adm.p);
}

long long squared_pattern(const Csr& A, int* out_ptr, int* out_idx, cudaStream_t s) {
    const int n = A.n, G = grid_for(n);
    DBuf<long long> cnt(n + 1, s), off(n + 1, s);
    UA_LAUNCH(k_sq_count, G, 256, 0, s, A, cnt.p);
    UA_CK(cudaMemsetAsync(cnt.p + n, 0, sizeof(long long), s));
    exclusive_scan(cnt.p, off.p, n + 1, s);
    long long total = 0;
    UA_CK(cudaMemcpyAsync(&total, off.p + n, sizeof(long long), cudaMemcpyDeviceToHost, s));
    UA_CK(cudaStreamSynchronize(s));
    DBuf<unsigned long long> keys(std::max(total, 1ll), s), sorted(std::max(total, 1ll), s), uniq(std::max(total, 1ll), s);
    UA_LAUNCH(k_sq_expand, G, 256, 0, s, A, off.p, keys.p);
    size_t tmp = 0;
    UA_CK(cub::DeviceRadixSort::SortKeys(nullptr, tmp, keys.p, sorted.p, (int)total, 0, 64, s));
    DBuf<char> t(tmp, s);
    UA_CK(cub::DeviceRadixSort::SortKeys(t.p, tmp, keys.p, sorted.p, (int)total, 0, 64, s));
    DBuf<int> nu(1, s);
    tmp = 0;
    UA_CK(cub::DeviceSelect::Unique(nullptr, tmp, sorted.p, uniq.p, nu.p, (int)total, s));
    DBuf<char> t2(tmp, s);
    UA_CK(cub::DeviceSelect::Unique(t2.p, tmp, sorted.p, uniq.p, nu.p, (int)total, s));
    int h_nu = 0;
    UA_CK(cudaMemcpyAsync(&h_nu, nu.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    UA_CK(cudaStreamSynchronize(s));
    squared_pattern_finish(n, uniq.p, h_nu, out_ptr, out_idx, s);
    return h_nu;
}

__global__ void k_sq_rows(int n, const unsigned long long* u, int m, int* ptr, int* idx) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < m; t += gridDim.x * blockDim.x) {
        const int r = (int)(u[t] >> 32);
        if (idx) idx[t] = (int)(u[t] & 0xffffffffu);
        const int rp = t == 0 ? -1 : (int)(u[t - 1] >> 32);
        for (int q = rp + 1; q <= r; ++q) ptr[q] = t;
        if (t == m - 1)
            for (int q = r + 1; q <= n; ++q) ptr[q] = m;
    }
}
void squared_pattern_finish(int n, const unsigned long long* uniq, int m, int* out_ptr, int* out_idx, cudaStream_t s) {
    if (m == 0) {
        UA_CK(cudaMemsetAsync(out_ptr, 0, sizeof(int) * (n + 1), s));
        return;
    }
    UA_LAUNCH(k_sq_rows, grid_for(m), 256, 0, s, n, uniq, m, out_ptr, out_idx);
}

void galerkin_table(const Csr& A, const int* v2a, int nc, int* out_ptr, int* out_col, double* out_val,
                    long long* nnz_c, cudaStream_t s) {
    DBuf<int> agg_ptr(nc + 1, s), members(std::max(A.n, 1), s);
    build_members(A.n, nc, v2a, agg_ptr.p, members.p, s);
    DBuf<int> rp, ci;
    DBuf<double> av;
    long long m = device_galerkin(A, v2a, nc, agg_ptr.p, members.p, rp, ci, av, s);
    *nnz_c = m;
    UA_CK(cudaMemcpyAsync(out_ptr, rp.p, sizeof(int) * (nc + 1), cudaMemcpyDeviceToDevice, s));
    if (out_col && m) {
        UA_CK(cudaMemcpyAsync(out_col, ci.p, sizeof(int) * m, cudaMemcpyDeviceToDevice, s));
        UA_CK(cudaMemcpyAsync(out_val, av.p, sizeof(double) * m, cudaMemcpyDeviceToDevice, s));
    }
    UA_CK(cudaStreamSynchronize(s));
}

}  // namespace uaamg
