// reshape.cu -- subgraph reshaping of aggregate pairs (Alg. 3, PAPER §3.3;
// reference U/reshaping.py:156-248, hooked into setup at
// U/hierarchy.py:141-144) as batched small dense problems on the GPU.
//
// Per sweep: the coarse edges (aggregate pairs joined by a fine edge) are
// sorted by (min id, max id) and matched greedily in that order (host, a
// linear pass: U/reshaping.py:226-232); every matched pair whose union has
// at most pair_cap vertices is one CTA of k_reshape_pairs:
//   * the union's local Laplacian A^ (U/reshaping.py:55-73), the smoother
//     error matrix S = I - M^-1 A^ (U/_dense.py:43-52) and the pseudo-inverse
//     A^+ (cyclic Jacobi eigensolver; cut 1e-12 lambda_max, U/_dense.py:8-16)
//     in shared memory;
//   * every balanced split (|V1| = floor(n/2), vertex 0 on side 1 for even n,
//     itertools.combinations order: U/reshaping.py:160-183) is unranked by a
//     thread, kept if both sides are connected (bitmask BFS), and scored by
//     the rank-one trace of W = S' A^ Q S A^+ (U/reshaping.py:121-141):
//     with y = A^ w, u = S' y, z = A^+ u, W = u z' / (w'y), and the
//     reference's rank_one_trace (first k with |W_kk| > 1e-12 max|W|:
//     tr = |W_:k|^2 / W_kk);
//   * the winner is the maximal |T|^2, ties to the earliest split in
//     enumeration order (the reference keeps the incumbent unless strictly
//     larger).  Values within 1e-10 relative are treated as ties: the
//     reference's own choice among mathematically tied splits depends on its
//     BLAS rounding (tests/test_gpu_reshape.py).
// Then the aggregates are renumbered by their smallest member
// (U/aggregation.py:248-257).
#include <cub/cub.cuh>

#include <math_constants.h>

#include <vector>

#include "setup.h"

namespace uaamg {

namespace {

constexpr int kRsMax = 16;       // largest pair the kernel enumerates (reference DEFAULT_PAIR_CAP)
constexpr int kRsThreads = 256;

__device__ __forceinline__ long long binom(int n, int k) {
    if (k < 0 || k > n) return 0;
    long long r = 1;
    for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
    return r;
}

// k-subset of {0..n-1} with lexicographic rank r, as a bitmask
__device__ unsigned unrank(long long r, int n, int k) {
    unsigned mask = 0;
    int x = 0;
    for (int i = 0; i < k; ++i) {
        while (true) {
            const long long c = binom(n - x - 1, k - i - 1);
            if (c <= r) {
                r -= c;
                ++x;
            } else {
                break;
            }
        }
        mask |= 1u << x;
        ++x;
    }
    return mask;
}

__device__ bool connected(unsigned side, const unsigned* adj) {
    if (side == 0) return true;
    unsigned reach = side & (~side + 1u);  // lowest vertex
    while (true) {
        unsigned nx = reach;
        for (unsigned b = reach; b; b &= b - 1) nx |= adj[__ffs(b) - 1] & side;
        if (nx == reach) break;
        reach = nx;
    }
    return reach == side;
}

__global__ void __launch_bounds__(kRsThreads) k_reshape_pairs(Csr A, int npairs, const int2* pairs,
                                                              const int* agg_ptr, const int* members, int l1,
                                                              double omega, int cap, int* v2a_out, int* status) {
    __shared__ int mem[kRsMax];
    __shared__ unsigned adj[kRsMax];
    __shared__ double ah[kRsMax][kRsMax], S[kRsMax][kRsMax], V[kRsMax][kRsMax], E[kRsMax][kRsMax];
    __shared__ double Ap[kRsMax][kRsMax];
    __shared__ double rot[2];
    __shared__ int m_s;
    __shared__ double bt[kRsThreads];
    __shared__ long long br[kRsThreads];
    const int b = blockIdx.x;
    if (b >= npairs) return;
    const int t = threadIdx.x;
    const int gi = pairs[b].x, gj = pairs[b].y;
    if (t == 0) {
        // union members, ascending (two sorted member lists merged)
        int p = agg_ptr[gi], pe = agg_ptr[gi + 1], q = agg_ptr[gj], qe = agg_ptr[gj + 1];
        const int m = (pe - p) + (qe - q);
        m_s = m;
        if (m <= cap && m <= kRsMax) {
            int k = 0;  // the union's vertices in ascending order
            while (p < pe || q < qe) {
                if (q >= qe || (p < pe && members[p] < members[q])) mem[k++] = members[p++];
                else mem[k++] = members[q++];
            }
        }
    }
    __syncthreads();
    const int m = m_s;
    if (m > cap || m > kRsMax) {
        if (t == 0) status[b] = 1;  // PairTooLarge: skipped (U/reshaping.py:236-240)
        return;
    }
    for (int e = t; e < kRsMax * kRsMax; e += blockDim.x) (&ah[0][0])[e] = 0.0;
    __syncthreads();
    if (t == 0) {
        // local Laplacian of the induced subgraph (U/reshaping.py:61-71)
        for (int k = 0; k < m; ++k) {
            const int v = mem[k];
            for (int e = A.rp[v]; e < A.rp[v + 1]; ++e) {
                const int col = A.ci[e];
                if (col == v) continue;
                int kc = -1;
                for (int c = 0; c < m; ++c)
                    if (mem[c] == col) kc = c;
                if (kc < 0) continue;
                const double w = -A.av[e];
                ah[k][kc] = -w;
                ah[k][k] = __dadd_rn(ah[k][k], w);
            }
        }
        for (int k = 0; k < m; ++k) {
            unsigned a = 0;
            for (int c = 0; c < m; ++c)
                if (c != k && ah[k][c] != 0.0) a |= 1u << c;
            adj[k] = a;
        }
    }
    __syncthreads();
    // smoother error matrix S = I - M^-1 A^ (U/_dense.py:43-52)
    if (t < m) {
        const double d = ah[t][t];
        double mi;
        if (l1) {
            double rs = 0.0;
            for (int c = 0; c < m; ++c) rs += fabs(ah[t][c]);
            mi = d + (rs - fabs(d));
        } else {
            mi = d / omega;
        }
        for (int c = 0; c < m; ++c) S[t][c] = (t == c ? 1.0 : 0.0) - ah[t][c] / mi;
        if (!(mi > 0.0)) status[b] = 3;  // non-positive smoother diagonal in the local problem
    }
    // symmetric copy for the eigensolver, V = I
    for (int e = t; e < m * m; e += blockDim.x) {
        const int i = e / m, j = e % m;
        E[i][j] = (ah[i][j] + ah[j][i]) / 2.0;
        V[i][j] = i == j ? 1.0 : 0.0;
    }
    __syncthreads();
    // cyclic Jacobi: rotation (p, q) computed by thread 0, applied by all
    for (int sw = 0; sw < 30; ++sw) {
        double off = 0.0, tot = 0.0;
        if (t == 0) {
            for (int i = 0; i < m; ++i)
                for (int j = 0; j < m; ++j) {
                    tot += E[i][j] * E[i][j];
                    if (i != j) off += E[i][j] * E[i][j];
                }
            rot[0] = off;
            rot[1] = tot;
        }
        __syncthreads();
        if (!(rot[0] > 1e-32 * rot[1])) break;
        __syncthreads();
        for (int p = 0; p < m; ++p)
            for (int q = p + 1; q < m; ++q) {
                if (t == 0) {
                    const double apq = E[p][q];
                    if (fabs(apq) < 1e-300) {
                        rot[0] = 1.0;
                        rot[1] = 0.0;
                    } else {
                        const double th = (E[q][q] - E[p][p]) / (2.0 * apq);
                        const double tt = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
                        const double c = 1.0 / sqrt(tt * tt + 1.0);
                        rot[0] = c;
                        rot[1] = tt * c;
                    }
                }
                __syncthreads();
                const double c = rot[0], s = rot[1];
                if (s != 0.0) {
                    // E <- J' E J, V <- V J  (rows / columns p, q)
                    if (t < m) {
                        const double ep = E[t][p], eq = E[t][q];
                        E[t][p] = c * ep - s * eq;
                        E[t][q] = s * ep + c * eq;
                    }
                    __syncthreads();
                    if (t < m) {
                        const double ep = E[p][t], eq = E[q][t];
                        E[p][t] = c * ep - s * eq;
                        E[q][t] = s * ep + c * eq;
                        const double vp = V[t][p], vq = V[t][q];
                        V[t][p] = c * vp - s * vq;
                        V[t][q] = s * vp + c * vq;
                    }
                }
                __syncthreads();
            }
    }
    // A^+ = V diag(1/lambda, lambda > 1e-12 lambda_max) V'
    __shared__ double lmax;
    if (t == 0) {
        double mx = -1e300;
        for (int k = 0; k < m; ++k) mx = fmax(mx, E[k][k]);
        lmax = mx;
    }
    __syncthreads();
    const double cut = 1e-12 * fmax(lmax, 0.0);
    for (int e = t; e < m * m; e += blockDim.x) {
        const int i = e / m, j = e % m;
        double s = 0.0;
        for (int k = 0; k < m; ++k)
            if (E[k][k] > cut) s += V[i][k] * (1.0 / E[k][k]) * V[j][k];
        Ap[i][j] = s;
    }
    __syncthreads();
    // balanced splits (U/reshaping.py:160-183)
    const int half = m / 2;
    const bool even = (m % 2) == 0;
    const long long ncand = even ? binom(m - 1, half - 1) : binom(m, half);
    const unsigned all = (m == 32) ? 0xffffffffu : ((1u << m) - 1u);
    double amax = 0.0;
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j) amax = fmax(amax, fabs(ah[i][j]));
    // |T|^2 of split rank r (the reference's rank_one_trace may be negative);
    // -inf: not a candidate (a side is disconnected)
    const double kNone = -CUDART_INF;
    auto score = [&](long long r) -> double {
        const unsigned s1 = even ? (1u | (unrank(r, m - 1, half - 1) << 1)) : unrank(r, m, half);
        const unsigned s2 = all & ~s1;
        if (!connected(s1, adj) || !connected(s2, adj)) return kNone;
        const int n1 = __popc(s1), n2 = m - n1;
        double w[kRsMax], y[kRsMax], u[kRsMax];
        for (int k = 0; k < m; ++k) w[k] = ((s1 >> k) & 1) ? 1.0 / n1 : -1.0 / n2;
        double waw = 0.0;
        for (int i = 0; i < m; ++i) {
            double a = 0.0;
            for (int k = 0; k < m; ++k) a += ah[i][k] * w[k];
            y[i] = a;
            waw += w[i] * a;
        }
        if (!(waw > 1e-14 * fmax(amax, 1.0))) return kNone;  // zero-energy coarse vector (disconnected union)
        double umax = 0.0, uu = 0.0;
        for (int i = 0; i < m; ++i) {
            double a = 0.0;
            for (int k = 0; k < m; ++k) a += S[k][i] * y[k];
            u[i] = a;
            umax = fmax(umax, fabs(a));
            uu += a * a;
        }
        // rank_one_trace (U/reshaping.py:105-118) of W = u z' / waw, z = A^+ u
        double zmax = 0.0;
        for (int i = 0; i < m; ++i) {
            double a = 0.0;
            for (int k = 0; k < m; ++k) a += Ap[i][k] * u[k];
            y[i] = a;  // z
            zmax = fmax(zmax, fabs(a));
        }
        const double scale = umax * zmax / waw;
        if (scale == 0.0) return 0.0;
        for (int k = 0; k < m; ++k) {
            const double wkk = u[k] * y[k] / waw;
            if (fabs(wkk) > 1e-12 * scale) return (uu * (y[k] / waw) * (y[k] / waw)) / wkk;
        }
        return 0.0;
    };
    // pass 1: the maximum; pass 2: the earliest split within 1e-10 of it
    double best = kNone;
    for (long long r = t; r < ncand; r += blockDim.x) best = fmax(best, score(r));
    bt[t] = best;
    __syncthreads();
    __shared__ double tmax_s;
    if (t == 0) {
        double tm = kNone;
        for (int k = 0; k < (int)blockDim.x; ++k) tm = fmax(tm, bt[k]);
        tmax_s = tm;
    }
    __syncthreads();
    const double tmax = tmax_s;
    long long first = -1;
    if (tmax > kNone)
        for (long long r = t; r < ncand; r += blockDim.x) {
            const double v = score(r);
            if (v > kNone && v >= tmax - 1e-10 * fabs(tmax)) {
                first = r;
                break;
            }
        }
    br[t] = first;
    __syncthreads();
    if (t == 0) {
        long long win = -1;
        for (int k = 0; k < (int)blockDim.x; ++k)
            if (br[k] >= 0 && (win < 0 || br[k] < win)) win = br[k];
        if (win < 0) {
            status[b] = 2;  // DisconnectedPair: no balanced connected split (U/reshaping.py:204-205)
        } else {
            const unsigned s1 = even ? (1u | (unrank(win, m - 1, half - 1) << 1)) : unrank(win, m, half);
            for (int k = 0; k < m; ++k) v2a_out[mem[k]] = ((s1 >> k) & 1) ? gi : gj;
        }
    }
}

// keys of coarse edges (gi < gj); others UINT64_MAX
__global__ void k_coarse_edge_keys(Csr A, const int* v2a, unsigned long long nc, unsigned long long* key) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += gridDim.x * blockDim.x) {
        const unsigned long long gi = (unsigned)v2a[i];
        for (int e = A.rp[i]; e < A.rp[i + 1]; ++e) {
            const unsigned long long gj = (unsigned)v2a[A.ci[e]];
            key[e] = gi < gj ? gi * nc + gj : ~0ull;
        }
    }
}
__global__ void k_min_member(int n, const int* v2a, int* mn) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) atomicMin(mn + v2a[v], v);
}
__global__ void k_iota_i(int n, int* v) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) v[i] = i;
}
__global__ void k_scatter_newid(int nc, const int* order, int* new_id) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nc; k += gridDim.x * blockDim.x) new_id[order[k]] = k;
}
__global__ void k_apply_newid(int n, const int* new_id, int* v2a) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) v2a[v] = new_id[v2a[v]];
}
int gsz(long long n) { return std::max(1, std::min(cdiv(n, 256), 4 * kNumSMs)); }

}  // namespace

// U/reshaping.py:215-248 on the device; v2a (n) is updated in place and
// seeds (nc) receives the smallest member of every aggregate.  Returns the
// number of pairs skipped for exceeding pair_cap.
int device_reshape_sweep(const Csr& A, int nc, int* v2a, int* seeds, int l1, double omega, int sweeps, int pair_cap,
                         cudaStream_t s) {
    if (pair_cap > kRsMax)
        throw Error(UAAMG_EUNSUPPORTED, "reshape pair_cap > 16 (exhaustive enumeration limit of the kernel)");
    const int n = A.n;
    int skipped = 0;
    const long long nnz = std::max(A.nnz, 1);
    for (int sw = 0; sw < sweeps; ++sw) {
        // coarse edges, sorted by (min id, max id), unique
        DBuf<unsigned long long> key(nnz, s), key2(nnz, s), uniq(nnz, s);
        DBuf<int> nuniq(1, s);
        UA_LAUNCH(k_coarse_edge_keys, gsz(n), 256, 0, s, A, v2a, (unsigned long long)nc, key.p);
        {
            size_t tmp = 0;
            UA_CK(cub::DeviceRadixSort::SortKeys(nullptr, tmp, key.p, key2.p, A.nnz, 0, 64, s));
            DBuf<char> tt(tmp, s);
            UA_CK(cub::DeviceRadixSort::SortKeys(tt.p, tmp, key.p, key2.p, A.nnz, 0, 64, s));
            tmp = 0;
            UA_CK(cub::DeviceSelect::Unique(nullptr, tmp, key2.p, uniq.p, nuniq.p, A.nnz, s));
            DBuf<char> t2(tmp, s);
            UA_CK(cub::DeviceSelect::Unique(t2.p, tmp, key2.p, uniq.p, nuniq.p, A.nnz, s));
        }
        int nu = 0;
        UA_CK(cudaMemcpyAsync(&nu, nuniq.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        UA_CK(cudaStreamSynchronize(s));
        std::vector<unsigned long long> edges(nu);
        if (nu) UA_CK(cudaMemcpyAsync(edges.data(), uniq.p, sizeof(unsigned long long) * nu, cudaMemcpyDeviceToHost, s));
        UA_CK(cudaStreamSynchronize(s));
        // greedy maximal matching in edge order (U/reshaping.py:226-231)
        std::vector<char> matched(nc, 0);
        std::vector<int2> pairs;
        for (unsigned long long e : edges) {
            if (e == ~0ull) break;  // sentinel block (no coarse edge)
            const int gi = (int)(e / (unsigned long long)nc), gj = (int)(e % (unsigned long long)nc);
            if (matched[gi] || matched[gj]) continue;
            matched[gi] = matched[gj] = 1;
            pairs.push_back(make_int2(gi, gj));
        }
        const int np = (int)pairs.size();
        if (np > 0) {
            DBuf<int> agg_ptr(nc + 1, s), members(n, s), out(n, s), status(np, s);
            DBuf<int2> dp(np, s);
            build_members(n, nc, v2a, agg_ptr.p, members.p, s);
            UA_CK(cudaMemcpyAsync(dp.p, pairs.data(), sizeof(int2) * np, cudaMemcpyHostToDevice, s));
            UA_CK(cudaMemcpyAsync(out.p, v2a, sizeof(int) * n, cudaMemcpyDeviceToDevice, s));
            UA_CK(cudaMemsetAsync(status.p, 0, sizeof(int) * np, s));
            UA_LAUNCH(k_reshape_pairs, np, kRsThreads, 0, s, A, np, dp.p, agg_ptr.p, members.p, l1, omega, pair_cap,
                      out.p, status.p);
            std::vector<int> st(np);
            UA_CK(cudaMemcpyAsync(st.data(), status.p, sizeof(int) * np, cudaMemcpyDeviceToHost, s));
            UA_CK(cudaStreamSynchronize(s));
            // pairs are processed in matching order by the reference: its
            // first failing pair decides the error
            for (int k = 0; k < np; ++k) {
                if (st[k] == 3) throw Error(UAAMG_EINVAL, "non-positive smoother diagonal in local problem");
                if (st[k] == 2) throw Error(UAAMG_EINVAL, "no balanced connected split exists");
                if (st[k] == 1) ++skipped;
            }
            UA_CK(cudaMemcpyAsync(v2a, out.p, sizeof(int) * n, cudaMemcpyDeviceToDevice, s));
        }
        // renumber by smallest member (U/aggregation.py:248-257)
        DBuf<int> mn(nc, s), order(nc, s), mn2(nc, s), iota(nc, s), nid(nc, s);
        UA_CK(cudaMemsetAsync(mn.p, 0x7f, sizeof(int) * nc, s));
        UA_LAUNCH(k_min_member, gsz(n), 256, 0, s, n, v2a, mn.p);
        UA_LAUNCH(k_iota_i, gsz(nc), 256, 0, s, nc, iota.p);
        size_t tmp = 0;
        UA_CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, mn.p, mn2.p, iota.p, order.p, nc, 0, 32, s));
        DBuf<char> tt(tmp, s);
        UA_CK(cub::DeviceRadixSort::SortPairs(tt.p, tmp, mn.p, mn2.p, iota.p, order.p, nc, 0, 32, s));
        UA_LAUNCH(k_scatter_newid, gsz(nc), 256, 0, s, nc, order.p, nid.p);
        UA_LAUNCH(k_apply_newid, gsz(n), 256, 0, s, n, nid.p, v2a);
        UA_CK(cudaMemcpyAsync(seeds, mn2.p, sizeof(int) * nc, cudaMemcpyDeviceToDevice, s));
        UA_CK(cudaStreamSynchronize(s));
    }
    return skipped;
}

}  // namespace uaamg
