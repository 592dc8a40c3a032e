// ops.cuh -- recorded solve operations for the persistent coarse engine.
//
// The host-side solve plan (runtime.cu, mirroring U/solvers.py:128-187)
// issues every operation through an Exec.  In recording mode each operation
// becomes an Op: a kind tag naming the functor types plus the functors'
// bytes.  The engine (engine.cu) switches on the kind and runs the SAME
// functor code the standalone kernels run, as one phase of a persistent
// cooperative kernel.  The X-macro lists below are the single source of the
// kind numbering for both sides.
#pragma once
#include <cstring>

#include "solve_ops.cuh"

namespace uaamg {

// dense coarsest solve x = Minv b (U/hierarchy.py:56-65)
struct DenseArgs {
    const double* M;
    const double* b;
    double* x;
    const int* g;
    int n;
};

//   X(kind, Src, Epi, Unit)
#define UA_ENGINE_CSR_OPS(X)                  \
    X(1, SrcPre1, EpiResid, false)            \
    X(2, SrcVec, EpiResid, false)             \
    X(3, SrcZero, EpiResid, false)            \
    X(4, SrcVec, EpiStoreG, true)             \
    X(5, SrcUp, EpiSweep, false)              \
    X(6, SrcVec, EpiSweep, false)             \
    X(7, SrcDir, EpiDirFcg, false)            \
    X(8, SrcUp, EpiSweepBeta, false)          \
    X(9, SrcVec, EpiSweepBeta, false)         \
    X(10, SrcVec, EpiRestrictBegin, true)     \
    X(11, SrcPre1, EpiResidSum, false)        \
    X(12, SrcVec, EpiResidSum, false)         \
    X(13, SrcZero, EpiResidSum, false)
//   X(kind, Body)
#define UA_ENGINE_MAP_OPS(X) \
    X(20, BodyXpre1)         \
    X(21, BodyProl)          \
    X(22, BodyFcgBegin)      \
    X(23, BodyBeta)          \
    X(24, BodyFcgUpd)        \
    X(25, BodyFcgProj)       \
    X(26, BodySum)           \
    X(27, BodySub)           \
    X(28, BodyCompat)
constexpr int kOpDense = 40;

constexpr int kOpPay = 224;

struct Op {
    int kind = 0;
    int n = 0;          // rows (CSR) / items (map)
    int small = 0;      // engine: runs on the first cluster only (cluster barriers)
    int sync_before = 0;  // engine: full grid barrier first (after a run of small ops)
    Csr A;              // CSR operand (CSR kinds)
    Groups G;
    alignas(16) unsigned char pay[kOpPay];
};

template <class Src, class Epi, bool Unit>
struct CsrKind {
    static constexpr int v = -1;
};
template <class Body>
struct MapKind {
    static constexpr int v = -1;
};
#define UA_CSR_KIND(k, S, E, U)              \
    template <>                              \
    struct CsrKind<S, E, U> {                \
        static constexpr int v = k;          \
    };
#define UA_MAP_KIND(k, B)                    \
    template <>                              \
    struct MapKind<B> {                      \
        static constexpr int v = k;          \
    };
UA_ENGINE_CSR_OPS(UA_CSR_KIND)
UA_ENGINE_MAP_OPS(UA_MAP_KIND)
#undef UA_CSR_KIND
#undef UA_MAP_KIND

template <class Src, class Epi>
struct CsrPay {
    Src src;
    Epi epi;
};

template <class Src, class Epi, bool Unit>
inline void record_csr(std::vector<Op>& rec, const Csr& A, const Groups& G, const Src& src, const Epi& epi) {
    constexpr int k = CsrKind<Src, Epi, Unit>::v;
    if (k < 0) throw Error(UAAMG_EUNSUPPORTED, "operation has no engine form");
    static_assert(sizeof(CsrPay<Src, Epi>) <= kOpPay, "op payload too large");
    Op op;
    op.kind = k;
    op.n = G.n;
    op.A = A;
    op.G = G;
    CsrPay<Src, Epi> p{src, epi};
    std::memcpy(op.pay, &p, sizeof(p));
    rec.push_back(op);
}

template <class Body>
inline void record_map(std::vector<Op>& rec, int n, const Body& body) {
    constexpr int k = MapKind<Body>::v;
    if (k < 0) throw Error(UAAMG_EUNSUPPORTED, "operation has no engine form");
    static_assert(sizeof(Body) <= kOpPay, "op payload too large");
    Op op;
    op.kind = k;
    op.n = n;
    std::memcpy(op.pay, &body, sizeof(body));
    rec.push_back(op);
}

inline void record_dense(std::vector<Op>& rec, const DenseArgs& d) {
    Op op;
    op.kind = kOpDense;
    op.n = d.n;
    std::memcpy(op.pay, &d, sizeof(d));
    rec.push_back(op);
}

}  // namespace uaamg
