// engine.h -- persistent coarse-level K-cycle engine (internal).
//
// Below a row-count threshold every level of the K-cycle is latency-bound:
// kernels of a few microseconds of work each, hundreds per NPCG iteration
// (level l is visited 2^l times).  The engine runs the whole recursion
// below a given level -- cycle() / _inner_fcg() of U/solvers.py:128-187 --
// inside ONE cooperative launch.  The host solve plan is recorded once into
// an op list (ops.cuh: the same functors the standalone kernels run); the
// engine interprets it with a grid barrier between phases.  Reductions are
// per-CTA partials that every CTA folds in the same fixed order after the
// barrier, so every CTA computes bit-identical scalars and flags and takes
// identical gate decisions; gated-off ops cost no barrier.
#pragma once
#include "ops.cuh"

namespace uaamg {

constexpr int kEngThreads = 512;  // one CTA per SM
constexpr int kEngK = 2;          // max values per reduction

struct EngineArgs {
    const Op* ops = nullptr;
    int nops = 0;
    const int* gate = nullptr;   // entry gate (nullptr: on); off -> no-op
    double* partials = nullptr;  // 2 tiers x 2 slots x kEngK x grid
    unsigned* bar = nullptr;     // [0] arrivals, [1] generation
    unsigned long long* prof = nullptr;  // diagnostics: globaltimer at each op start (nops + 1)
    int csize = 0;               // cluster size (set by launch_engine)
};

// default engine entry: first level with at most this many rows (0: the
// engine is off by default -- per-op latency in the persistent kernel does
// not yet beat graph-replayed launches of the group kernel on B200)
constexpr long long kEngDefaultRows = 0;
// ops on at most this many rows run on one cluster (cluster barriers)
constexpr int kEngSmallRows = 65536;

int engine_grid();
int engine_cluster();
void launch_engine(const EngineArgs& a, cudaStream_t s);

}  // namespace uaamg
