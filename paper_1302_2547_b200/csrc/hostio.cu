// hostio.cu -- host <-> device transfers of the reference-layout host arrays
// (the drop-in's input path: U/sparse.py SparseMatrix holds int64 indptr /
// indices and float64 data in pageable numpy memory; the device layout is
// int32 / int32 / float64).
//
// A pageable cudaMemcpy moves ~10 GB/s and a host-side int64 -> int32 pass
// costs another full sweep, so both are replaced by a pipeline: a persistent
// ring of pinned staging chunks, filled by OpenMP worker threads (copy, or
// narrow int64 -> int32 while copying), each chunk handed to the copy engine
// as soon as it is full while the threads fill the next one.
#include <omp.h>

#include <cstring>
#include <mutex>

#include "common.cuh"

namespace uaamg {
extern thread_local std::string g_last_error;

namespace {
constexpr size_t kChunk = 8u << 20;  // bytes per staging chunk
constexpr int kRing = 4;
struct Ring {
    char* buf[kRing] = {};
    cudaEvent_t ev[kRing] = {};
    bool init = false;
};
std::mutex g_ring_mu;
Ring g_ring[kMaxDevices];

Ring& ring(int dev) {
    Ring& R = g_ring[dev];
    if (!R.init) {
        for (int k = 0; k < kRing; ++k) {
            UA_CK(cudaHostAlloc((void**)&R.buf[k], kChunk, cudaHostAllocPortable));
            UA_CK(cudaEventCreateWithFlags(&R.ev[k], cudaEventDisableTiming));
        }
        R.init = true;
    }
    return R;
}
int threads() {
    static const int t = [] {
        const int c = omp_get_num_procs();
        const char* e = getenv("UAAMG_STAGE_THREADS");  // A/B diagnostics
        const int cap = e ? atoi(e) : 8;
        return c < 2 ? 1 : (c > cap ? cap : c);
    }();
    return t;
}

// dst_elem == src_elem: copy; 8 -> 4: narrow int64 -> int32
void fill(char* dst, const char* src, size_t count, int se, int de) {
    if (se == de) {
        const size_t bytes = count * se, per = (bytes + threads() - 1) / threads();
#pragma omp parallel for num_threads(threads()) schedule(static)
        for (int t = 0; t < threads(); ++t) {
            const size_t b0 = per * t;
            if (b0 < bytes) std::memcpy(dst + b0, src + b0, std::min(per, bytes - b0));
        }
    } else {
        const long long* s = reinterpret_cast<const long long*>(src);
        int* d = reinterpret_cast<int*>(dst);
#pragma omp parallel for num_threads(threads()) schedule(static)
        for (long long i = 0; i < (long long)count; ++i) d[i] = (int)s[i];
    }
}
}  // namespace

void staged_h2d(void* dst, const void* src, size_t count, int se, int de, cudaStream_t s) {
    if (!count) return;
    if (!(se == de || (se == 8 && de == 4))) throw Error(UAAMG_EINVAL, "unsupported element sizes");
    std::lock_guard<std::mutex> lk(g_ring_mu);
    Ring& R = ring(cur_dev());
    const size_t per_chunk = kChunk / se;  // elements per chunk (source side bounds the staging)
    size_t done = 0;
    for (int k = 0; done < count; ++k) {
        const int slot = k % kRing;
        const size_t m = std::min(per_chunk, count - done);
        UA_CK(cudaEventSynchronize(R.ev[slot]));  // the copy engine released this chunk
        fill(R.buf[slot], static_cast<const char*>(src) + done * se, m, se, de);
        UA_CK(cudaMemcpyAsync(static_cast<char*>(dst) + done * de, R.buf[slot], m * de, cudaMemcpyHostToDevice, s));
        UA_CK(cudaEventRecord(R.ev[slot], s));
        done += m;
    }
    for (int k = 0; k < kRing; ++k) UA_CK(cudaEventSynchronize(R.ev[k]));  // the source may be reused
}

void staged_d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (!bytes) return;
    std::lock_guard<std::mutex> lk(g_ring_mu);
    Ring& R = ring(cur_dev());
    // chunk k lands in the ring while chunk k-1 is copied out by the threads
    size_t done = 0;
    int k = 0;
    size_t prev_off = 0, prev_m = 0;
    int prev_slot = -1;
    while (done < bytes || prev_slot >= 0) {
        int slot = -1;
        size_t m = 0;
        if (done < bytes) {
            slot = k % kRing;
            m = std::min(kChunk, bytes - done);
            UA_CK(cudaMemcpyAsync(R.buf[slot], static_cast<const char*>(src) + done, m, cudaMemcpyDeviceToHost, s));
            UA_CK(cudaEventRecord(R.ev[slot], s));
        }
        if (prev_slot >= 0) {
            UA_CK(cudaEventSynchronize(R.ev[prev_slot]));
            fill(static_cast<char*>(dst) + prev_off, R.buf[prev_slot], prev_m, 1, 1);
        }
        prev_slot = slot;
        prev_off = done;
        prev_m = m;
        done += m;
        ++k;
    }
}

}  // namespace uaamg

using namespace uaamg;

extern "C" {

int uaamg_h2d(void* dst, const void* src, int64_t count, int src_elem, int dst_elem, void* stream) {
    try {
        staged_h2d(dst, src, (size_t)count, src_elem, dst_elem, (cudaStream_t)stream);
        return UAAMG_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    }
}

int uaamg_d2h(void* dst, const void* src, int64_t bytes, void* stream) {
    try {
        staged_d2h(dst, src, (size_t)bytes, (cudaStream_t)stream);
        return UAAMG_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    }
}

}  // extern "C"
