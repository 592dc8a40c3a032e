// dist.h -- row-partitioned (multi-rank) setup and solve (internal).
//
// SURVEY.md §8e.  Level 0 is split into P contiguous row blocks; every rank
// holds only its rows (global column indices) and computes only its rows.
// Coarse levels inherit the partition without repartitioning: aggregates are
// numbered by ascending seed (U/aggregation.py:199-203), so the aggregates
// whose seed lies in rank q's rows are a contiguous block of the next level.
// Levels smaller than `shard_rows` are gathered and replicated: every rank
// builds (bit-identically) and runs them whole with the single-device path.
//
// Data plane: every array a peer reads lives in a per-rank ARENA.  A kernel
// reads element k of a distributed array from the rank that owns k --
// locally for own rows, by a peer load for halo entries (on an 8xB200 box an
// NVLink load from the CUDA-IPC-mapped peer arena; the "halo exchange" is the
// gather itself, fused into the consuming kernel).  Ranks are ordered by a
// device-side flag barrier between phases.  Virtual ranks (rank < 0) run all
// P ranks in one process on one device, launched rank by rank in one stream
// (stream order is the barrier): the partition-invariance harness.
#pragma once
#include "launch.cuh"
#include "runtime.h"

namespace uaamg {

constexpr int kSlotK = 2;  // max values per cross-rank reduction (Epi::K)

// ---------------------------------------------------------------- comm
struct Comm {
    int P = 1;
    int rank = -1;            // -1: virtual ranks (all in this process)
    std::vector<int> mine;    // ranks this process computes
    cudaStream_t s = 0;
    int dev = 0;
    // per rank: arena base (own, peer-mapped, or -- virtual -- all own)
    std::vector<char*> base;
    size_t cap = 0;                 // arena bytes (same on every rank)
    std::vector<size_t> lo, hi;     // per local rank: persistent bump (up), scratch bump (down)
    DBuf<unsigned> epoch;           // this rank's barrier count (device: barriers are graph-capturable)
    int ndir = 0, nval = 0;         // rolling directory / value slot cursors
    DBuf<unsigned*> flag_tab;       // P barrier flag lines
    bool connected = false;
    int users = 0;                  // live hierarchies on the arena (the bumps reset when the last goes)
    static constexpr size_t kHeader = 1 << 20;  // directory + values + flags
    static constexpr int kDirSlots = 4096, kValSlots = 4096;
    static constexpr size_t kDirOff = 0, kValOff = 8 * kDirSlots, kFlagOff = 16 * kDirSlots;

    bool virt() const { return rank < 0; }
    ~Comm();
    // create the arenas of this process's ranks (multi-process: then
    // exchange IPC handles and connect)
    void create(int P_, int rank_, size_t bytes, cudaStream_t st);
    void connect(const void* handles);  // multi-process: P cudaIpcMemHandle_t
    void connect_virtual();
    // device barrier across ranks (no-op for virtual ranks: stream order);
    // gate: skipped when *gate == 0 (identically on every rank: a gated-off
    // NPCG iteration runs no barrier anywhere)
    void barrier(const int* gate = nullptr);
    void host_barrier() {
        barrier();
        UA_CK(cudaStreamSynchronize(s));
    }
    // arena allocation for local rank r (persistent or per-level scratch)
    void* alloc_bytes(int r, size_t bytes, bool scratch);
    template <class T>
    T* alloc(int r, size_t count, bool scratch = false) {
        return static_cast<T*>(alloc_bytes(r, count * sizeof(T), scratch));
    }
    void reset_scratch();
    void release_user() {
        if (--users == 0)
            for (int r : mine) { lo[r] = kHeader; hi[r] = cap; }
    }
    // every rank's pointer for one buffer per local rank (collective)
    std::vector<std::vector<void*>> tables(const std::vector<std::vector<void*>>& local);
    template <class T>
    std::vector<T*> table(const std::vector<T*>& local) {
        std::vector<void*> v(local.begin(), local.end());
        auto t = tables({v});
        std::vector<T*> out(P);
        for (int q = 0; q < P; ++q) out[q] = static_cast<T*>(t[0][q]);
        return out;
    }
    // every rank's value (collective): local[r] for r in mine
    std::vector<long long> allgather(const std::vector<long long>& local);
    long long allsum(const std::vector<long long>& local) {
        long long t = 0;
        for (long long v : allgather(local)) t += v;
        return t;
    }
};

// peer accessor of a distributed array: element k lives on rank owner(k) at
// tab[owner(k)][k] (tables hold base pointers shifted by the owner's first row)
template <class T>
struct DV {
    Part pt;
    T* tab[kMaxRanks];
    __device__ __forceinline__ T& operator[](int k) const { return tab[pt.owner(k)][k]; }
};

// peer accessor of a row-partitioned CSR (rows of rank q: rp[q][k], shifted)
struct DCsr {
    Part pt;
    const int* rp[kMaxRanks];
    const int* ci[kMaxRanks];
    const double* av[kMaxRanks];
};

// ---------------------------------------------------------------- hierarchy
struct DRank {            // one rank's share of a sharded level
    int a = 0, n = 0;     // own rows [a, a + n)
    long long nnz = 0;
    int* rp = nullptr;    // n + 1 local offsets, stored so that rp - a is 16-byte aligned modulo 4 rows
    int* rps = nullptr;   // shifted: rps[i] for global row i
    int* ci = nullptr;    // global column indices
    double* av = nullptr;
    int* v2a = nullptr;   // own rows -> global coarse index
    int* seeds = nullptr; // own seeds (ascending global fine indices) = coarse rows [ca, ca + nca)
    int nseeds = 0;
    int* mptr = nullptr;  // members of aggregates [mbase, mbase + mcount): rows of mptr, global fine ids
    int* mem = nullptr;
    int mbase = 0, mcount = 0;
};
struct DLevel {
    int n = 0;            // global rows
    long long nnz = 0;    // global nonzeros
    Part pt{};
    int nc = 0;           // global coarse rows (0: last sharded level has not aggregated yet)
    Part cpt{};
    std::vector<DRank> r;  // [P]
    DCsr A{};              // peer tables
};

struct DistHier {
    std::shared_ptr<Comm> C;
    ~DistHier() {
        rep.reset();
        lv.clear();
        if (C) C->release_user();
    }
    std::vector<DLevel> lv;                  // sharded levels 0 .. Ls-1
    std::unique_ptr<uaamg_hierarchy> rep;    // replicated levels Ls .. (every rank)
    bool singular = false;
    double setup_seconds = 0, grid_complexity = 1, operator_complexity = 1;
    int Ls() const { return (int)lv.size(); }
    int nlevels() const { return Ls() + (rep ? (int)rep->levels.size() : 0); }
    int level_n(int l) const { return l < Ls() ? lv[l].n : rep->levels[l - Ls()]->n; }
    long long level_nnz(int l) const { return l < Ls() ? lv[l].nnz : rep->levels[l - Ls()]->nnz; }
};

// level 0 on the local ranks: rp/ci/av[k] = rows of rank mine[k]
std::unique_ptr<DistHier> dist_setup(std::shared_ptr<Comm> C, int n, const int* bounds,
                                     const std::vector<const int*>& rp, const std::vector<const int*>& ci,
                                     const std::vector<const double*>& av, const std::vector<long long>& nnz,
                                     const uaamg_setup_params& P, long long shard_rows);

Part level0_part(int n, int P);
// renumbering by ascending seed (U/aggregation.py:199-203): rank q's
// aggregates are [b[q], b[q+1]) with b the exclusive scan of the per-rank
// seed counts (host-only)
Part coarse_bounds(const long long* counts, int P);

}  // namespace uaamg
