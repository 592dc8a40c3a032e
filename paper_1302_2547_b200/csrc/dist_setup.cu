// dist_setup.cu -- the communicator and the row-partitioned setup
// (U/hierarchy.py:120-153 with U/aggregation.py:144-203 and
// K/numba_backend.py:145-273 sharded by rows).
//
// Per sharded level and rank (own rows only; entries of other ranks are
// read from their arenas through DV / DCsr peer accessors):
//   aggregation  the multi-pass parallel aggregation as phase kernels --
//                scores, max-hop, select, max-hop, claim, admission
//                fixpoint, commit -- each reading its depth-1 halo (state,
//                score, hop maxima, owner, admitted flag) from the owners;
//                pass / fixpoint control from per-rank counts all-gathered
//                by the host after a barrier.  Same semantics as the
//                single-device kernels (kernels_setup.cu), so the
//                aggregation is bit-identical for any rank count.
//   renumbering  seeds (centers and leftovers) counted per rank, counts
//                all-gathered, exclusive scan: rank q's aggregates are the
//                contiguous block [off_q, off_q + cnt_q) (U/aggregation.py:
//                199-203); v2a[j] = new id of j's seed (peer read, the seed
//                is within distance 2).
//   members      every rank sorts (aggregate, vertex) keys of its rows and
//                publishes them; the owner of each aggregate pulls its block
//                from every rank (an all-to-all through peer memory).
//   Galerkin     the owner of aggregate I pulls the rows of I's members
//                (remote rows included), maps columns to coarse indices
//                (v2a of the column's owner) and emits (I, J, a) in the
//                reference's order (members ascending, entries ascending);
//                a stable radix sort by (I, J) and a sequential segmented
//                sum reproduce galerkin_coo (K/numba_backend.py:145-172):
//                stable mergesort + in-order sums, exact zeros dropped --
//                bit-identical for any weights.
// Below `shard_rows` the next level is gathered (every rank copies every
// rank's rows) and the remaining levels are set up by the single-device
// path on every rank (replicated, bit-identical).
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <numeric>
#include <type_traits>

#include "dist.h"

namespace uaamg {

// ================================================================ comm
// cross-device barrier: count it on this rank (device counter, so captured
// graphs replay correctly), publish the count into every rank's flag line,
// then wait until every rank has published it into ours.  gate == 0: the
// whole NPCG iteration is gated off on every rank alike -- no barrier.
__global__ void k_dist_barrier(unsigned* const* flags, int P, int rank, unsigned* ctr, const int* gate) {
    if (gate && *(const volatile int*)gate == 0) return;
    const unsigned epoch = ++*ctr;
    __threadfence_system();  // this rank's earlier writes (own and peer) first
    for (int q = 0; q < P; ++q) *(volatile unsigned*)(flags[q] + 32 * rank) = epoch;
    __threadfence_system();
    const volatile unsigned* mine = flags[rank];
    const long long t0 = clock64();
    for (int q = 0; q < P; ++q)
        while ((int)(mine[32 * q] - epoch) < 0) {
            __nanosleep(64);
            if (clock64() - t0 > (1ll << 36)) __trap();  // a rank died: fail loudly
        }
    __threadfence_system();
}

Comm::~Comm() {
    if (!connected && base.empty()) return;
    cudaStreamSynchronize(s);
    for (int q = 0; q < (int)base.size(); ++q) {
        if (!base[q]) continue;
        if (virt() || q == rank) cudaFree(base[q]);
        else cudaIpcCloseMemHandle(base[q]);
    }
}

void Comm::create(int P_, int rank_, size_t bytes, cudaStream_t st) {
    if (P_ < 1 || P_ > kMaxRanks) throw Error(UAAMG_EINVAL, "ranks must be in [1, 8]");
    if (rank_ >= P_) throw Error(UAAMG_EINVAL, "rank out of range");
    P = P_;
    rank = rank_;
    s = st;
    dev = cur_dev();
    mine.clear();
    if (rank < 0) for (int q = 0; q < P; ++q) mine.push_back(q);
    else mine.push_back(rank);
    cap = ((bytes + kHeader + 4095) / 4096) * 4096;
    base.assign(P, nullptr);
    lo.assign(P, kHeader);
    hi.assign(P, cap);
    for (int r : mine) {
        UA_CK(cudaMalloc(&base[r], cap));
        UA_CK(cudaMemset(base[r], 0, kHeader));
    }
}

void Comm::connect(const void* handles) {
    const auto* hs = static_cast<const cudaIpcMemHandle_t*>(handles);
    for (int q = 0; q < P; ++q) {
        if (q == rank) continue;
        void* p = nullptr;
        UA_CK(cudaIpcOpenMemHandle(&p, hs[q], cudaIpcMemLazyEnablePeerAccess));
        base[q] = static_cast<char*>(p);
    }
    std::vector<unsigned*> fl(P);
    for (int q = 0; q < P; ++q) fl[q] = reinterpret_cast<unsigned*>(base[q] + kFlagOff);
    flag_tab.alloc(P, s);
    epoch.alloc(1, s);
    UA_CK(cudaMemsetAsync(epoch.p, 0, sizeof(unsigned), s));
    UA_CK(cudaMemcpyAsync(flag_tab.p, fl.data(), sizeof(unsigned*) * P, cudaMemcpyHostToDevice, s));
    UA_CK(cudaStreamSynchronize(s));
    connected = true;
    host_barrier();
}

void Comm::connect_virtual() { connected = true; }

void Comm::barrier(const int* gate) {
    if (virt()) return;
    UA_LAUNCH(k_dist_barrier, 1, 1, 0, s, flag_tab.p, P, rank, epoch.p, gate);
}

void* Comm::alloc_bytes(int r, size_t bytes, bool scratch) {
    const size_t b = ((bytes + 64 + 255) / 256) * 256;  // 64 B tail slack (TMA granules)
    if (lo[r] + b > hi[r])
        throw Error(UAAMG_ECUDA, "distributed arena exhausted (" + std::to_string(cap >> 20) +
                                     " MiB): raise arena_bytes");
    if (scratch) {
        hi[r] -= b;
        return base[r] + hi[r];
    }
    void* p = base[r] + lo[r];
    lo[r] += b;
    return p;
}

void Comm::reset_scratch() {
    for (int r : mine) hi[r] = cap;
}

std::vector<std::vector<void*>> Comm::tables(const std::vector<std::vector<void*>>& local) {
    const int m = (int)local.size();
    std::vector<std::vector<void*>> out(m, std::vector<void*>(P, nullptr));
    if (virt()) {
        for (int k = 0; k < m; ++k)
            for (int q = 0; q < P; ++q) out[k][q] = local[k][q];
        return out;
    }
    // publish offsets into this rank's directory, barrier, read the peers'
    if (ndir + m > kDirSlots) ndir = 0;  // rolling (slots are reused only after later barriers)
    const int slot0 = ndir;
    ndir += m;
    std::vector<long long> offs(m);
    for (int k = 0; k < m; ++k)
        offs[k] = local[k][rank] ? (long long)(static_cast<char*>(local[k][rank]) - base[rank]) : -1;
    UA_CK(cudaMemcpyAsync(base[rank] + kDirOff + 8 * slot0, offs.data(), 8 * m, cudaMemcpyHostToDevice, s));
    host_barrier();
    std::vector<long long> peer(m);
    for (int q = 0; q < P; ++q) {
        UA_CK(cudaMemcpy(peer.data(), base[q] + kDirOff + 8 * slot0, 8 * m, cudaMemcpyDeviceToHost));
        for (int k = 0; k < m; ++k) out[k][q] = peer[k] < 0 ? nullptr : base[q] + peer[k];
    }
    return out;
}

std::vector<long long> Comm::allgather(const std::vector<long long>& local) {
    std::vector<long long> out(P, 0);
    if (virt()) {
        for (int q = 0; q < P; ++q) out[q] = local[q];
        return out;
    }
    const int slot = nval;
    nval = (nval + 1) % kValSlots;
    long long v = local[rank];
    UA_CK(cudaMemcpyAsync(base[rank] + kValOff + 8 * slot, &v, 8, cudaMemcpyHostToDevice, s));
    host_barrier();
    for (int q = 0; q < P; ++q)
        UA_CK(cudaMemcpy(&out[q], base[q] + kValOff + 8 * slot, 8, cudaMemcpyDeviceToHost));
    return out;
}

// ================================================================ kernels
__device__ __forceinline__ uint64_t d_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static uint64_t h_pass_base(uint64_t seed, int64_t pass_idx) {
    uint64_t z = seed ^ (0xA0761D6478BD642Full * (uint64_t)(pass_idx + 1));
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ bool dkey_gt(double sa, int ia, double sb, int ib) {
    return sa > sb || (sa == sb && ia < ib);
}
static int g1(long long n) { return std::max(1, std::min(cdiv(n, 256), 8 * kNumSMs)); }

// v_i = d_i + ((i mod 12) + u_i) / 12 (K/numba_backend.py:100-111), own rows
__global__ void kd_scores(int a, int n, const int* rps, uint64_t base, double* s) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const int i = a + t;
        const uint64_t z = d_mix64(d_mix64(base + (uint64_t)i * 0x9E3779B97F4A7C15ull));
        const double u = __dmul_rn((double)(z >> 11), 1.0 / 9007199254740992.0);
        const double deg = (double)(rps[i + 1] - rps[i]);
        s[t] = __dadd_rn(deg, __ddiv_rn(__dadd_rn((double)(i % 12), u), 12.0));
    }
}

// state: 0 unprocessed, 1 center of this pass, 2 processed (kernels_setup.cu)
// Every row phase below runs rows of at most kDLong entries thread-per-row
// and the longer ("hub") rows of the level warp-per-row from a list (rows
// of coarse levels can span thousands of columns); all phases are
// order-free (key maxima, flags), so the split does not change results.
constexpr int kDLong = 64;

__global__ void kd_long_rows(int n, const int* rp, int* list, int* cnt) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
        if (rp[t + 1] - rp[t] > kDLong) list[atomicAdd(cnt, 1)] = t;
}

__device__ __forceinline__ void dwarp_keymax(double& s, int& i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double s2 = __shfl_xor_sync(0xffffffffu, s, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, i, o);
        if (i2 >= 0 && (i < 0 || dkey_gt(s2, i2, s, i))) { s = s2; i = i2; }
    }
}

// key maximum of f(e) = (score, index or -1) over entries [e0, e1):
// sequential in one thread, or (warp = true) strided over the 32 lanes and
// reduced (the maximum is unique: keys are distinct)
template <bool Warp, class F>
__device__ __forceinline__ void dkeymax(int e0, int e1, F&& f, double& bs, int& bi) {
    bs = 0.0;
    bi = -1;
    const int lane = Warp ? (threadIdx.x & 31) : 0;
    for (int e = e0 + lane; e < e1; e += Warp ? 32 : 1) {
        double v;
        int j;
        f(e, v, j);
        if (j >= 0 && (bi < 0 || dkey_gt(v, j, bs, bi))) { bs = v; bi = j; }
    }
    if (Warp) dwarp_keymax(bs, bi);
}

// runs body(t, warp) for every own row t: short rows by one thread each,
// long rows (list) by one warp each
template <class B>
__device__ __forceinline__ void drows(int n, const int* rps, int a, const int* longs, int nlong, B&& body) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
        if (rps[a + t + 1] - rps[a + t] <= kDLong) body(t, std::false_type{});
    const int warps = (gridDim.x * blockDim.x) >> 5;
    for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nlong; w += warps) body(longs[w], std::true_type{});
}

// hop 1 over own rows k: max key over j in row k with (mode 0: st != 2, mode 1: st == 1)
__global__ void kd_hop1(int a, int n, const int* rps, const int* ci, const int* longs, int nlong,
                        DV<const uint8_t> st, DV<const double> sc, int mode, double* ms, int* mi) {
    drows(n, rps, a, longs, nlong, [&](int t, auto warp) {
        constexpr bool W = decltype(warp)::value;
        const int k = a + t;
        double bs;
        int bi;
        dkeymax<W>(rps[k], rps[k + 1], [&](int e, double& v, int& j) {
            j = __ldg(ci + e);
            const uint8_t sj = st[j];
            if (mode == 0 ? (sj == 2) : (sj != 1)) { j = -1; return; }
            v = sc[j];
        }, bs, bi);
        if (!W || (threadIdx.x & 31) == 0) {
            ms[t] = bs;
            mi[t] = bi;
        }
    });
}

// best (ms[k], mi[k]) over k in row i
template <bool W>
__device__ __forceinline__ void dhop2(const int* rps, const int* ci, int i, const DV<const double>& ms,
                                      const DV<const int>& mi, double& bs, int& bi) {
    dkeymax<W>(rps[i], rps[i + 1], [&](int e, double& v, int& c) {
        const int k = __ldg(ci + e);
        c = mi[k];
        if (c >= 0) v = ms[k];
    }, bs, bi);
}

// select (K/numba_backend.py:175-193) on own rows
__global__ void kd_select(int a, int n, const int* rps, const int* ci, const int* longs, int nlong, const double* sc,
                          uint8_t* st, DV<const double> ms, DV<const int> mi, int* cnt) {
    int local = 0;
    drows(n, rps, a, longs, nlong, [&](int t, auto warp) {
        constexpr bool W = decltype(warp)::value;
        if (st[t] != 0) return;
        const int i = a + t;
        double bs;
        int bi;
        dhop2<W>(rps, ci, i, ms, mi, bs, bi);
        if ((!W || (threadIdx.x & 31) == 0) && (bi < 0 || bi == i || dkey_gt(sc[t], i, bs, bi))) {
            st[t] = 1;
            ++local;
        }
    });
    local = __reduce_add_sync(0xffffffffu, local);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(cnt, local);
}

// claim (K/numba_backend.py:196-220) on own rows
__global__ void kd_claim(int a, int n, const int* rps, const int* ci, const int* longs, int nlong, const double* sc,
                         const uint8_t* st, DV<const double> ms, DV<const int> mi, int* owner) {
    drows(n, rps, a, longs, nlong, [&](int t, auto warp) {
        constexpr bool W = decltype(warp)::value;
        const int j = a + t;
        const uint8_t sj = st[t];
        if (sj == 1) { owner[t] = j; return; }
        if (sj == 2) { owner[t] = -1; return; }
        double bs;
        int bi;
        dhop2<W>(rps, ci, j, ms, mi, bs, bi);
        if (!W || (threadIdx.x & 31) == 0) owner[t] = (bi >= 0 && !(bs < sc[t])) ? bi : -1;
    });
}

// uncapped admission (K/numba_backend.py:235-273): the fixpoint of "j is
// admitted if row(j) holds an admitted vertex of its own center"
__global__ void kd_admit_init(int n, const uint8_t* st, uint8_t* adm) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) adm[t] = (st[t] == 1);
}
__global__ void kd_admit_step(int a, int n, const int* rps, const int* ci, const int* longs, int nlong,
                              const int* owner_loc, uint8_t* adm_loc, DV<const uint8_t> adm, DV<const int> owner,
                              int* changed) {
    int local = 0;
    drows(n, rps, a, longs, nlong, [&](int t, auto warp) {
        constexpr bool W = decltype(warp)::value;
        const int j = a + t;
        const int c = owner_loc[t];
        if (c < 0 || c == j || adm_loc[t]) return;
        bool f = false;
        const int lane = W ? (threadIdx.x & 31) : 0;
        for (int e = rps[j] + lane; e < rps[j + 1]; e += W ? 32 : 1) {
            const int nb = __ldg(ci + e);
            if (*(const volatile uint8_t*)&adm[nb] && owner[nb] == c) {
                f = true;
                break;
            }
        }
        if (W) f = __any_sync(0xffffffffu, f);
        if (f && (!W || lane == 0)) {
            adm_loc[t] = 1;
            local = 1;
        }
    });
    if (__any_sync(0xffffffffu, local) && (threadIdx.x & 31) == 0) atomicOr(changed, 1);
}
__global__ void kd_commit(int n, uint8_t* st, const int* owner, const uint8_t* adm, int* seed_of, int* remaining) {
    int local = 0;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const uint8_t sj = st[t];
        if (sj == 1 || (sj == 0 && adm[t])) {
            seed_of[t] = owner[t];
            st[t] = 2;
        } else if (sj == 0) {
            ++local;
        }
    }
    local = __reduce_add_sync(0xffffffffu, local);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(remaining, local);
}
// leftovers become singletons (U/aggregation.py:195-198); seed flags
__global__ void kd_leftover(int a, int n, const uint8_t* st, int* seed_of, int* flag) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        if (st[t] != 2) seed_of[t] = a + t;
        flag[t] = seed_of[t] == a + t;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) flag[n] = 0;
}
// new index of own seeds (exclusive scan + rank offset), own seed list
__global__ void kd_newid(int a, int n, const int* flag, const int* scan, int off, int* nid, int* seeds) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
        if (flag[t]) {
            nid[t] = off + scan[t];
            seeds[scan[t]] = a + t;
        }
}
__global__ void kd_v2a(int n, const int* seed_of, DV<const int> nid, int* v2a) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) v2a[t] = nid[seed_of[t]];
}

// members: (aggregate << 32 | vertex) per own row
__global__ void kd_member_keys(int a, int n, const int* v2a, unsigned long long* key) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
        key[t] = ((unsigned long long)(unsigned)v2a[t] << 32) | (unsigned)(a + t);
}
// bnd[q] = first key whose aggregate belongs to coarse rank >= q
__global__ void kd_bounds(const unsigned long long* key, int n, Part cpt, int* bnd) {
    const int q = threadIdx.x;
    if (q > cpt.P) return;
    if (q == cpt.P) { bnd[q] = n; return; }
    const unsigned long long k0 = (unsigned long long)(unsigned)cpt.b[q] << 32;
    int lo = 0, hi = n;
    while (lo < hi) {
        const int m = (lo + hi) >> 1;
        if (key[m] < k0) lo = m + 1; else hi = m;
    }
    bnd[q] = lo;
}
// members CSR from sorted keys of aggregates [mbase, mbase + mcount)
__global__ void kd_members(const unsigned long long* key, int m, int mbase, int* cnt, int* mem) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < m; t += gridDim.x * blockDim.x) {
        const int I = (int)(key[t] >> 32) - mbase;
        mem[t] = (int)(key[t] & 0xffffffffu);
        atomicAdd(cnt + I, 1);
    }
}

__device__ __forceinline__ void drow(const DCsr& A, int k, int& q, int& e0, int& e1) {
    q = A.pt.owner(k);
    e0 = A.rp[q][k];
    e1 = A.rp[q][k + 1];
}
// Galerkin emission: entry counts per member row
__global__ void kd_gal_len(int m, const int* mem, DCsr A, int* len) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < m; t += gridDim.x * blockDim.x) {
        int q, e0, e1;
        drow(A, mem[t], q, e0, e1);
        len[t] = e1 - e0;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) len[m] = 0;
}
// (I_local << 32 | J, a) for every entry of every member row, members in
// order (aggregate-major, ascending vertex), entries in row order
__global__ void kd_gal_emit(int nagg, const int* mptr, const int* mem, const int* off, DCsr A, DV<const int> v2a,
                            unsigned long long* key, double* val) {
    const int lane = threadIdx.x & 31;
    const int warps = (gridDim.x * blockDim.x) >> 5;
    for (int I = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; I < nagg; I += warps) {
        for (int t = mptr[I]; t < mptr[I + 1]; ++t) {
            int q, e0, e1;
            drow(A, mem[t], q, e0, e1);
            const int o = off[t] - e0;
            for (int e = e0 + lane; e < e1; e += 32) {
                const int k = __ldg(A.ci[q] + e);
                key[o + e] = ((unsigned long long)(unsigned)I << 32) | (unsigned)v2a[k];
                val[o + e] = __ldg(A.av[q] + e);
            }
        }
    }
}
// segment heads of the sorted keys
__global__ void kd_heads(const unsigned long long* key, long long m, int* head) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < m; t += (long long)gridDim.x * blockDim.x)
        head[t] = (t == 0 || key[t] != key[t - 1]) ? 1 : 0;
}
__global__ void kd_head_pos(long long m, const int* head, const int* hscan, int* pos) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < m; t += (long long)gridDim.x * blockDim.x)
        if (head[t]) pos[hscan[t]] = (int)t;
}
// sequential in-order sum of each (I, J) segment (K/numba_backend.py:160-170)
__global__ void kd_seg_sum(int nseg, long long m, const int* pos, const unsigned long long* key, const double* val,
                           double* sum, int* keep, int* rowcnt) {
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < nseg; g += gridDim.x * blockDim.x) {
        const long long b = pos[g], e = g + 1 < nseg ? pos[g + 1] : m;
        double acc = 0.0;
        for (long long t = b; t < e; ++t) acc = __dadd_rn(acc, val[t]);
        sum[g] = acc;
        keep[g] = acc != 0.0;
        if (acc != 0.0) atomicAdd(rowcnt + (int)(key[b] >> 32), 1);
    }
}
__global__ void kd_seg_place(int nseg, const int* pos, const unsigned long long* key, const double* sum,
                             const int* keep, const int* kscan, int* ci, double* av) {
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < nseg; g += gridDim.x * blockDim.x)
        if (keep[g]) {
            ci[kscan[g]] = (int)(key[pos[g]] & 0xffffffffu);
            av[kscan[g]] = sum[g];
        }
}
// level-0 singular detection pieces (U/hierarchy.py:112-117): max|a|, max|A 1|
__global__ void kd_singular(int n, const int* rp, const double* av, unsigned long long* out) {
    double ma = 0.0, mr = 0.0;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        double r = 0.0;
        for (int e = rp[t]; e < rp[t + 1]; ++e) {
            const double v = __ldg(av + e);
            r = __dadd_rn(r, v);
            ma = fmax(ma, fabs(v));
        }
        mr = fmax(mr, fabs(r));
    }
    ma = block_max(ma);
    mr = block_max(mr);
    if (threadIdx.x == 0) {
        atomicMax(out, (unsigned long long)__double_as_longlong(ma));
        atomicMax(out + 1, (unsigned long long)__double_as_longlong(mr));
    }
}
// gathered rows: row pointers of rank q's block shifted by its entry offset
__global__ void kd_shift_rp(int n, const int* src, int add, int* dst) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t <= n; t += gridDim.x * blockDim.x) dst[t] = src[t] + add;
}

// ================================================================ host driver
namespace {

template <class T>
void scan_excl(const T* in, T* out, long long n, cudaStream_t s) {
    size_t tmp = 0;
    UA_CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, s));
    DBuf<char> t(tmp, s);
    UA_CK(cub::DeviceScan::ExclusiveSum(t.p, tmp, in, out, n, s));
}

int key_bits(unsigned long long v) {
    int b = 1;
    while (b < 64 && (v >> b)) ++b;
    return b;
}

void sort_keys(unsigned long long*& k, unsigned long long*& kalt, long long m, int end_bit, cudaStream_t s) {
    cub::DoubleBuffer<unsigned long long> db(k, kalt);
    size_t tmp = 0;
    UA_CK(cub::DeviceRadixSort::SortKeys(nullptr, tmp, db, m, 0, end_bit, s));
    DBuf<char> t(tmp, s);
    UA_CK(cub::DeviceRadixSort::SortKeys(t.p, tmp, db, m, 0, end_bit, s));
    k = db.Current();
    kalt = db.Alternate();
}

struct Setup {
    std::shared_ptr<Comm> C;
    const uaamg_setup_params& P;
    cudaStream_t s;
    DistHier& H;
    Comm& c() { return *C; }

    // local rows of a sharded level stored in the arena (rp with the
    // alignment pad, see DRank)
    void place_rows(DRank& R, int r, const int* rp_src, const int* ci_src, const double* av_src) {
        int* rpb = c().alloc<int>(r, (size_t)R.n + 8);
        R.rp = rpb + (R.a & 3);
        R.rps = R.rp - R.a;
        R.ci = c().alloc<int>(r, std::max<long long>(R.nnz, 1));
        R.av = c().alloc<double>(r, std::max<long long>(R.nnz, 1));
        UA_CK(cudaMemcpyAsync(R.rp, rp_src, sizeof(int) * (R.n + 1), cudaMemcpyDeviceToDevice, s));
        if (R.nnz) {
            UA_CK(cudaMemcpyAsync(R.ci, ci_src, sizeof(int) * R.nnz, cudaMemcpyDeviceToDevice, s));
            UA_CK(cudaMemcpyAsync(R.av, av_src, sizeof(double) * R.nnz, cudaMemcpyDeviceToDevice, s));
        }
    }

    void publish_csr(DLevel& L) {
        std::vector<void*> rp(c().P), ci(c().P), av(c().P);
        for (int r : c().mine) { rp[r] = L.r[r].rp; ci[r] = L.r[r].ci; av[r] = L.r[r].av; }
        auto t = c().tables({rp, ci, av});
        L.A.pt = L.pt;
        for (int q = 0; q < c().P; ++q) {
            L.A.rp[q] = static_cast<const int*>(t[0][q]) - L.pt.b[q];
            L.A.ci[q] = static_cast<const int*>(t[1][q]);
            L.A.av[q] = static_cast<const double*>(t[2][q]);
        }
    }

    template <class T>
    DV<T> dv(const Part& pt, const std::vector<void*>& tab) {
        DV<T> d{};
        d.pt = pt;
        for (int q = 0; q < c().P; ++q) d.tab[q] = static_cast<T*>(tab[q]) - pt.b[q];
        return d;
    }

    // multi-pass aggregation of sharded level l (uncapped); fills v2a,
    // seeds, nc, cpt.  Returns the global coarse size.
    int aggregate(int l) {
        DLevel& L = H.lv[l];
        Comm& C_ = c();
        const int P_ = C_.P;
        std::vector<void*> vst(P_), vs(P_), vms(P_), vmi(P_), vown(P_), vadm(P_), vseed(P_), vnid(P_);
        std::vector<int*> cnt(P_);
        for (int r : C_.mine) {
            const size_t n = std::max(L.r[r].n, 1);
            vst[r] = C_.alloc<uint8_t>(r, n, true);
            vs[r] = C_.alloc<double>(r, n, true);
            vms[r] = C_.alloc<double>(r, n, true);
            vmi[r] = C_.alloc<int>(r, n, true);
            vown[r] = C_.alloc<int>(r, n, true);
            vadm[r] = C_.alloc<uint8_t>(r, n, true);
            vseed[r] = C_.alloc<int>(r, n, true);
            vnid[r] = C_.alloc<int>(r, n, true);
            cnt[r] = C_.alloc<int>(r, 8, true);
            UA_CK(cudaMemsetAsync(vst[r], 0, n, s));
            UA_CK(cudaMemsetAsync(vseed[r], 0xff, sizeof(int) * n, s));
        }
        // rows longer than kDLong (per local rank), processed warp-per-row
        std::vector<int*> longs(P_, nullptr);
        std::vector<int> nlong(P_, 0);
        for (int r : C_.mine) {
            const DRank& R = L.r[r];
            longs[r] = C_.alloc<int>(r, std::max(R.n, 1), true);
            DBuf<int> c1(1, s);
            UA_CK(cudaMemsetAsync(c1.p, 0, sizeof(int), s));
            UA_LAUNCH(kd_long_rows, g1(R.n), 256, 0, s, R.n, R.rp, longs[r], c1.p);
            UA_CK(cudaMemcpyAsync(&nlong[r], c1.p, sizeof(int), cudaMemcpyDeviceToHost, s));
            UA_CK(cudaStreamSynchronize(s));
        }
        auto T = C_.tables({vst, vs, vms, vmi, vown, vadm, vnid});
        const DV<const uint8_t> st = dv<const uint8_t>(L.pt, T[0]);
        const DV<const double> sc = dv<const double>(L.pt, T[1]);
        const DV<const double> ms = dv<const double>(L.pt, T[2]);
        const DV<const int> mi = dv<const int>(L.pt, T[3]);
        const DV<const int> own = dv<const int>(L.pt, T[4]);
        const DV<const uint8_t> adm = dv<const uint8_t>(L.pt, T[5]);
        const DV<const int> nid = dv<const int>(L.pt, T[6]);
        // host readback of one device int per local rank, all-gathered
        auto gather_count = [&](int slot) {
            std::vector<long long> v(P_, 0);
            for (int r : C_.mine) {
                int h = 0;
                UA_CK(cudaMemcpyAsync(&h, cnt[r] + slot, sizeof(int), cudaMemcpyDeviceToHost, s));
                UA_CK(cudaStreamSynchronize(s));
                v[r] = h;
            }
            return C_.allsum(v);
        };
        long long remaining = L.n;
        for (int pass = 0; pass < P.max_passes; ++pass) {
            if (remaining == 0) break;
            const uint64_t base = h_pass_base(P.seed, pass);
            for (int r : C_.mine) {
                const DRank& R = L.r[r];
                UA_CK(cudaMemsetAsync(cnt[r], 0, sizeof(int) * 8, s));
                UA_LAUNCH(kd_scores, g1(R.n), 256, 0, s, R.a, R.n, R.rps, base, (double*)vs[r]);
            }
            C_.barrier();
            for (int r : C_.mine) {
                const DRank& R = L.r[r];
                UA_LAUNCH(kd_hop1, g1(R.n), 256, 0, s, R.a, R.n, R.rps, R.ci, longs[r], nlong[r], st, sc, 0,
                          (double*)vms[r], (int*)vmi[r]);
            }
            C_.barrier();
            for (int r : C_.mine) {
                const DRank& R = L.r[r];
                UA_LAUNCH(kd_select, g1(R.n), 256, 0, s, R.a, R.n, R.rps, R.ci, longs[r], nlong[r], (const double*)vs[r],
                          (uint8_t*)vst[r],
                          ms, mi, cnt[r] + 0);
            }
            if (gather_count(0) == 0) break;  // (includes a barrier)
            for (int r : C_.mine) {
                const DRank& R = L.r[r];
                UA_LAUNCH(kd_hop1, g1(R.n), 256, 0, s, R.a, R.n, R.rps, R.ci, longs[r], nlong[r], st, sc, 1,
                          (double*)vms[r], (int*)vmi[r]);
            }
            C_.barrier();
            for (int r : C_.mine) {
                const DRank& R = L.r[r];
                UA_LAUNCH(kd_claim, g1(R.n), 256, 0, s, R.a, R.n, R.rps, R.ci, longs[r], nlong[r], (const double*)vs[r],
                          (const uint8_t*)vst[r], ms, mi, (int*)vown[r]);
                UA_LAUNCH(kd_admit_init, g1(R.n), 256, 0, s, R.n, (const uint8_t*)vst[r], (uint8_t*)vadm[r]);
            }
            C_.barrier();
            for (int it = 0;; ++it) {
                const int slot = 1 + (it & 1);
                for (int r : C_.mine) {
                    const DRank& R = L.r[r];
                    UA_CK(cudaMemsetAsync(cnt[r] + slot, 0, sizeof(int), s));
                    UA_LAUNCH(kd_admit_step, g1(R.n), 256, 0, s, R.a, R.n, R.rps, R.ci, longs[r], nlong[r], (const int*)vown[r],
                              (uint8_t*)vadm[r], adm, own, cnt[r] + slot);
                }
                if (gather_count(slot) == 0) break;
            }
            for (int r : C_.mine) {
                const DRank& R = L.r[r];
                UA_LAUNCH(kd_commit, g1(R.n), 256, 0, s, R.n, (uint8_t*)vst[r], (const int*)vown[r],
                          (const uint8_t*)vadm[r], (int*)vseed[r], cnt[r] + 3);
            }
            remaining = gather_count(3);
        }
        // leftovers, renumbering by ascending seed
        std::vector<int*> flag(P_), scan(P_);
        std::vector<long long> nseeds(P_, 0);
        for (int r : C_.mine) {
            DRank& R = L.r[r];
            flag[r] = C_.alloc<int>(r, (size_t)R.n + 1, true);
            scan[r] = C_.alloc<int>(r, (size_t)R.n + 1, true);
            UA_LAUNCH(kd_leftover, g1(R.n), 256, 0, s, R.a, R.n, (const uint8_t*)vst[r], (int*)vseed[r], flag[r]);
            scan_excl(flag[r], scan[r], (long long)R.n + 1, s);
            int h = 0;
            UA_CK(cudaMemcpyAsync(&h, scan[r] + R.n, sizeof(int), cudaMemcpyDeviceToHost, s));
            UA_CK(cudaStreamSynchronize(s));
            nseeds[r] = h;
        }
        const std::vector<long long> all = C_.allgather(nseeds);
        L.cpt = coarse_bounds(all.data(), P_);
        L.nc = L.cpt.b[P_];
        for (int r : C_.mine) {
            DRank& R = L.r[r];
            R.nseeds = (int)all[r];
            R.seeds = C_.alloc<int>(r, std::max(R.nseeds, 1));
            R.v2a = C_.alloc<int>(r, std::max(R.n, 1));
            UA_LAUNCH(kd_newid, g1(R.n), 256, 0, s, R.a, R.n, flag[r], scan[r], L.cpt.b[r], (int*)vnid[r], R.seeds);
        }
        C_.barrier();
        for (int r : C_.mine) {
            DRank& R = L.r[r];
            UA_LAUNCH(kd_v2a, g1(R.n), 256, 0, s, R.n, (const int*)vseed[r], nid, R.v2a);
        }
        C_.barrier();
        return L.nc;
    }

    // members CSR per rank: own aggregates, or (all = true) every aggregate
    void members(int l, bool all) {
        DLevel& L = H.lv[l];
        Comm& C_ = c();
        const int P_ = C_.P;
        std::vector<void*> vkey(P_), vbnd(P_);
        for (int r : C_.mine) {
            DRank& R = L.r[r];
            const size_t n = std::max(R.n, 1);
            auto* k = C_.alloc<unsigned long long>(r, n, true);
            DBuf<unsigned long long> alt(n, s);
            UA_LAUNCH(kd_member_keys, g1(R.n), 256, 0, s, R.a, R.n, R.v2a, k);
            unsigned long long* cur = k;
            unsigned long long* other = alt.p;
            sort_keys(cur, other, R.n, 64, s);
            if (cur != k) UA_CK(cudaMemcpyAsync(k, cur, sizeof(unsigned long long) * R.n, cudaMemcpyDeviceToDevice, s));
            vkey[r] = k;
            vbnd[r] = C_.alloc<int>(r, kMaxRanks + 1, true);
            UA_LAUNCH(kd_bounds, 1, 32, 0, s, k, R.n, L.cpt, (int*)vbnd[r]);
            UA_CK(cudaStreamSynchronize(s));  // alt is freed
        }
        auto T = C_.tables({vkey, vbnd});
        // host copies of every rank's bounds
        std::vector<std::vector<int>> bnd(P_, std::vector<int>(kMaxRanks + 1));
        for (int q = 0; q < P_; ++q)
            UA_CK(cudaMemcpy(bnd[q].data(), T[1][q], sizeof(int) * (kMaxRanks + 1), cudaMemcpyDeviceToHost));
        for (int r : C_.mine) {
            DRank& R = L.r[r];
            const int b0 = all ? 0 : r, b1 = all ? P_ : r + 1;  // coarse-rank blocks wanted
            long long m = 0;
            for (int q = 0; q < P_; ++q) m += bnd[q][b1] - bnd[q][b0];
            DBuf<unsigned long long> recv(std::max<long long>(m, 1), s), alt(std::max<long long>(m, 1), s);
            long long o = 0;
            for (int q = 0; q < P_; ++q) {
                const long long c0 = bnd[q][b0], c1 = bnd[q][b1];
                if (c1 > c0)
                    UA_CK(cudaMemcpyAsync(recv.p + o, static_cast<unsigned long long*>(T[0][q]) + c0,
                                          sizeof(unsigned long long) * (c1 - c0), cudaMemcpyDefault, s));
                o += c1 - c0;
            }
            unsigned long long* cur = recv.p;
            unsigned long long* other = alt.p;
            sort_keys(cur, other, m, 64, s);
            R.mbase = all ? 0 : L.cpt.b[r];
            R.mcount = all ? L.nc : L.cpt.b[r + 1] - L.cpt.b[r];
            DBuf<int> cntb((size_t)R.mcount + 1, s);
            UA_CK(cudaMemsetAsync(cntb.p, 0, sizeof(int) * (R.mcount + 1), s));
            R.mem = C_.alloc<int>(r, std::max<long long>(m, 1));
            R.mptr = C_.alloc<int>(r, (size_t)R.mcount + 1);
            UA_LAUNCH(kd_members, g1(m), 256, 0, s, cur, (int)m, R.mbase, cntb.p, R.mem);
            scan_excl(cntb.p, R.mptr, (long long)R.mcount + 1, s);
            UA_CK(cudaStreamSynchronize(s));
        }
        C_.barrier();  // peers' key blocks may be recycled after this
    }

    // Galerkin of own aggregates -> next level's rows on each rank
    void galerkin(int l, DLevel& N) {
        DLevel& L = H.lv[l];
        Comm& C_ = c();
        const int P_ = C_.P;
        std::vector<void*> vv2a(P_);
        for (int r : C_.mine) vv2a[r] = L.r[r].v2a;
        const DV<const int> v2a = dv<const int>(L.pt, C_.tables({vv2a})[0]);
        N.n = L.nc;
        N.pt = L.cpt;
        N.r.resize(P_);
        std::vector<long long> nnzs(P_, 0);
        for (int r : C_.mine) {
            DRank& R = L.r[r];
            DRank& Q = N.r[r];
            Q.a = L.cpt.b[r];
            Q.n = L.cpt.b[r + 1] - L.cpt.b[r];
            int nm = 0;
            UA_CK(cudaMemcpyAsync(&nm, R.mptr + R.mcount, sizeof(int), cudaMemcpyDeviceToHost, s));
            UA_CK(cudaStreamSynchronize(s));
            // own aggregates' members: the whole CSR (all = false), or the
            // block of this rank's aggregates (all = true)
            const int I0 = Q.a - R.mbase;
            int t0 = 0, t1 = nm;
            if (R.mbase != Q.a || R.mcount != Q.n) {
                UA_CK(cudaMemcpyAsync(&t0, R.mptr + I0, sizeof(int), cudaMemcpyDeviceToHost, s));
                UA_CK(cudaMemcpyAsync(&t1, R.mptr + I0 + Q.n, sizeof(int), cudaMemcpyDeviceToHost, s));
                UA_CK(cudaStreamSynchronize(s));
            }
            const int mm = t1 - t0;
            DBuf<int> len((size_t)mm + 1, s), off((size_t)mm + 1, s), lptr((size_t)Q.n + 1, s);
            UA_LAUNCH(kd_gal_len, g1(std::max(mm, 1)), 256, 0, s, mm, R.mem + t0, L.A, len.p);
            scan_excl(len.p, off.p, (long long)mm + 1, s);
            int ne = 0;
            UA_CK(cudaMemcpyAsync(&ne, off.p + mm, sizeof(int), cudaMemcpyDeviceToHost, s));
            // aggregate pointers relative to t0
            UA_LAUNCH(kd_shift_rp, g1(Q.n + 1), 256, 0, s, Q.n, R.mptr + I0, -t0, lptr.p);
            UA_CK(cudaStreamSynchronize(s));
            const long long E = std::max(ne, 1);
            DBuf<unsigned long long> key(E, s), kalt(E, s);
            DBuf<double> val(E, s), valt(E, s);
            UA_LAUNCH(kd_gal_emit, std::max(1, std::min(cdiv((long long)Q.n * 32, 256), 16 * kNumSMs)), 256, 0, s, Q.n, lptr.p,
                      R.mem + t0, off.p, L.A, v2a, key.p, val.p);
            // stable sort by (I, J): equal keys keep the reference's order
            cub::DoubleBuffer<unsigned long long> dk(key.p, kalt.p);
            cub::DoubleBuffer<double> dvv(val.p, valt.p);
            const int eb = 32 + key_bits((unsigned long long)std::max(Q.n, 1));
            size_t tmp = 0;
            UA_CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, dk, dvv, ne, 0, eb, s));
            {
                DBuf<char> t(tmp, s);
                UA_CK(cub::DeviceRadixSort::SortPairs(t.p, tmp, dk, dvv, ne, 0, eb, s));
            }
            const unsigned long long* sk = dk.Current();
            const double* sv = dvv.Current();
            DBuf<int> head(E + 1, s), hscan(E + 1, s);
            UA_LAUNCH(kd_heads, g1(E), 256, 0, s, sk, (long long)ne, head.p);
            UA_CK(cudaMemsetAsync(head.p + ne, 0, sizeof(int), s));
            scan_excl(head.p, hscan.p, (long long)ne + 1, s);
            int nseg = 0;
            UA_CK(cudaMemcpyAsync(&nseg, hscan.p + ne, sizeof(int), cudaMemcpyDeviceToHost, s));
            UA_CK(cudaStreamSynchronize(s));
            DBuf<int> pos(std::max(nseg, 1), s), keep(nseg + 1, s), kscan(nseg + 1, s), rowcnt((size_t)Q.n + 1, s);
            DBuf<double> sum(std::max(nseg, 1), s);
            UA_LAUNCH(kd_head_pos, g1(E), 256, 0, s, (long long)ne, head.p, hscan.p, pos.p);
            UA_CK(cudaMemsetAsync(rowcnt.p, 0, sizeof(int) * (Q.n + 1), s));
            UA_LAUNCH(kd_seg_sum, g1(std::max(nseg, 1)), 256, 0, s, nseg, (long long)ne, pos.p, sk, sv, sum.p, keep.p,
                      rowcnt.p);
            UA_CK(cudaMemsetAsync(keep.p + nseg, 0, sizeof(int), s));
            scan_excl(keep.p, kscan.p, (long long)nseg + 1, s);
            int nk = 0;
            UA_CK(cudaMemcpyAsync(&nk, kscan.p + nseg, sizeof(int), cudaMemcpyDeviceToHost, s));
            UA_CK(cudaStreamSynchronize(s));
            Q.nnz = nk;
            nnzs[r] = nk;
            int* rpb = C_.alloc<int>(r, (size_t)Q.n + 8);
            Q.rp = rpb + (Q.a & 3);
            Q.rps = Q.rp - Q.a;
            Q.ci = C_.alloc<int>(r, std::max(nk, 1));
            Q.av = C_.alloc<double>(r, std::max(nk, 1));
            scan_excl(rowcnt.p, Q.rp, (long long)Q.n + 1, s);
            UA_LAUNCH(kd_seg_place, g1(std::max(nseg, 1)), 256, 0, s, nseg, pos.p, sk, sum.p, keep.p, kscan.p, Q.ci,
                      Q.av);
            UA_CK(cudaStreamSynchronize(s));
        }
        N.nnz = C_.allsum(nnzs);
        publish_csr(N);
    }

    // every rank's rows of a sharded level, gathered into one local CSR
    void gather(const DLevel& L, DBuf<int>& rp, DBuf<int>& ci, DBuf<double>& av) {
        Comm& C_ = c();
        const int P_ = C_.P;
        std::vector<long long> nz(P_, 0);
        for (int r : C_.mine) nz[r] = L.r[r].nnz;
        const auto all = C_.allgather(nz);
        rp.alloc((size_t)L.n + 1, s);
        ci.alloc(std::max<long long>(L.nnz, 1), s);
        av.alloc(std::max<long long>(L.nnz, 1), s);
        long long o = 0;
        for (int q = 0; q < P_; ++q) {
            const int a = L.pt.b[q], n = L.pt.b[q + 1] - a;
            // L.A.rp[q] is shifted: rows [a, a + n] start at L.A.rp[q] + a
            UA_LAUNCH(kd_shift_rp, g1(n + 1), 256, 0, s, n, L.A.rp[q] + a, (int)o, rp.p + a);
            if (all[q]) {
                UA_CK(cudaMemcpyAsync(ci.p + o, L.A.ci[q], sizeof(int) * all[q], cudaMemcpyDefault, s));
                UA_CK(cudaMemcpyAsync(av.p + o, L.A.av[q], sizeof(double) * all[q], cudaMemcpyDefault, s));
            }
            o += all[q];
        }
        UA_CK(cudaStreamSynchronize(s));
        C_.barrier();  // nobody recycles rows a peer may still be copying
    }
};

}  // namespace

// level 0 of a row-partitioned setup (see dist.h)
std::unique_ptr<DistHier> dist_setup(std::shared_ptr<Comm> Cp, int n, const int* bounds,
                                     const std::vector<const int*>& rp, const std::vector<const int*>& ci,
                                     const std::vector<const double*>& av, const std::vector<long long>& nnz,
                                     const uaamg_setup_params& P, long long shard_rows) {
    Comm& C = *Cp;
    if (!C.connected) throw Error(UAAMG_EINVAL, "communicator is not connected");
    if (P.size_cap > 0) throw Error(UAAMG_EUNSUPPORTED, "sharded setup supports size_cap=None only");
    if (P.passes_per_level != 1) throw Error(UAAMG_EUNSUPPORTED, "sharded setup supports passes_per_level=1 only");
    if (P.reshape_sweeps > 0) throw Error(UAAMG_EUNSUPPORTED, "sharded setup supports reshape_sweeps=0 only");
    if (P.max_passes < 1) throw Error(UAAMG_EAGG, "max_passes must be >= 1");
    if (n <= 0) throw Error(UAAMG_EINVAL, "matrix must be non-empty");
    cudaStream_t s = C.s;
    if (C.users > 0) throw Error(UAAMG_EINVAL, "a hierarchy already lives on this communicator's arena");
    auto H = std::make_unique<DistHier>();
    H->C = Cp;
    ++C.users;
    cudaEvent_t e0, e1;
    UA_CK(cudaEventCreate(&e0));
    UA_CK(cudaEventCreate(&e1));
    UA_CK(cudaEventRecord(e0, s));
    Setup S{Cp, P, s, *H};
    // level 0: the caller's rows
    DLevel L0;
    L0.n = n;
    L0.pt.P = C.P;
    for (int q = 0; q <= kMaxRanks; ++q) L0.pt.b[q] = bounds[std::min(q, C.P)];
    for (int q = 0; q < C.P; ++q)
        if (L0.pt.b[q + 1] < L0.pt.b[q]) throw Error(UAAMG_EINVAL, "row bounds must be nondecreasing");
    if (L0.pt.b[0] != 0 || L0.pt.b[C.P] != n) throw Error(UAAMG_EINVAL, "row bounds must cover [0, n)");
    L0.r.resize(C.P);
    std::vector<long long> nz(C.P, 0);
    for (size_t k = 0; k < C.mine.size(); ++k) {
        const int r = C.mine[k];
        DRank& R = L0.r[r];
        R.a = L0.pt.b[r];
        R.n = L0.pt.b[r + 1] - R.a;
        R.nnz = nnz[k];
        nz[r] = R.nnz;
        S.place_rows(R, r, rp[k], ci[k], av[k]);
    }
    L0.nnz = C.allsum(nz);
    H->lv.push_back(std::move(L0));
    S.publish_csr(H->lv[0]);
    // singular (U/hierarchy.py:112-117): max over ranks of max|a| and max|A 1|
    if (P.singular < 0) {
        std::vector<long long> ma(C.P, 0), mr(C.P, 0);
        for (int r : C.mine) {
            const DRank& R = H->lv[0].r[r];
            DBuf<unsigned long long> mx(2, s);
            UA_CK(cudaMemsetAsync(mx.p, 0, 16, s));
            UA_LAUNCH(kd_singular, g1(R.n), 256, 0, s, R.n, R.rp, R.av, mx.p);
            unsigned long long h[2];
            UA_CK(cudaMemcpyAsync(h, mx.p, 16, cudaMemcpyDeviceToHost, s));
            UA_CK(cudaStreamSynchronize(s));
            ma[r] = (long long)h[0];
            mr[r] = (long long)h[1];
        }
        const auto A = C.allgather(ma), R = C.allgather(mr);
        double scale = 0, ax = 0;
        for (int q = 0; q < C.P; ++q) {  // non-negative doubles: bit order = value order
            double a, b;
            std::memcpy(&a, &A[q], 8);
            std::memcpy(&b, &R[q], 8);
            scale = std::max(scale, a);
            ax = std::max(ax, b);
        }
        H->singular = (H->lv[0].nnz == 0) || ax <= 1e-10 * scale;
    } else {
        H->singular = P.singular != 0;
    }
    // sharded levels while big enough (same stopping rule as U/hierarchy.py:133)
    const long long thr = std::max<long long>(shard_rows, (long long)P.n0 + 1);
    int nl = 0;  // levels so far (sharded)
    bool gather_now = !(n >= thr && P.max_levels > 1);
    while (!gather_now) {
        DLevel& L = H->lv[nl];
        const int nc = S.aggregate(nl);
        if (nc == L.n)
            throw Error(UAAMG_ESETUP, "aggregation stagnated at level " + std::to_string(nl) + ": " +
                                          std::to_string(L.n) + " vertices produced no coarsening");
        ++nl;  // level nl-1 now has an aggregation; level nl is its Galerkin product
        const bool next_sharded = nc >= thr && nl < P.max_levels - 1;
        S.members(nl - 1, !next_sharded);
        DLevel N;
        S.galerkin(nl - 1, N);
        C.reset_scratch();
        H->lv.push_back(std::move(N));
        // otherwise the next level is the first replicated one (the last
        // sharded level keeps the members of ALL its aggregates: every rank
        // restricts into the whole replicated level)
        if (!next_sharded) gather_now = true;
    }
    // gather the first replicated level and set up the rest on every rank
    DLevel G = std::move(H->lv.back());
    H->lv.pop_back();
    {
        DBuf<int> grp, gci;
        DBuf<double> gav;
        Setup S2{Cp, P, s, *H};
        S2.gather(G, grp, gci, gav);
        uaamg_setup_params Q = P;
        Q.max_levels = P.max_levels - (int)H->lv.size();
        Q.singular = H->singular ? 1 : 0;
        Q.borrow = 0;
        H->rep.reset(setup_impl(G.n, G.nnz, grp.p, gci.p, gav.p, Q, s, (int)H->lv.size()));
        UA_CK(cudaStreamSynchronize(s));
    }
    // the gathered level's arena rows are no longer needed by peers but stay
    // allocated (bump allocator); complexities over all levels
    UA_CK(cudaEventRecord(e1, s));
    UA_CK(cudaEventSynchronize(e1));
    float ms = 0;
    UA_CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    H->setup_seconds = ms * 1e-3;
    double sn = 0, snz = 0;
    for (int l = 0; l < H->nlevels(); ++l) {
        sn += H->level_n(l);
        snz += (double)H->level_nnz(l);
    }
    H->grid_complexity = sn / n;
    H->operator_complexity = snz / std::max<double>((double)H->level_nnz(0), 1.0);
    return H;
}

}  // namespace uaamg
