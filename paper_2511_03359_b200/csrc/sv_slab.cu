// Caching allocator for state slabs (host side).
//
// run_circuit allocates a 2^N state per call; at N = 33 that is a 128 GiB
// cudaMalloc + cudaFree per circuit (tens of ms of page-table work, and a
// device-wide synchronisation in cudaFree).  Freed slabs of >= 1 MiB are kept
// per device and handed back to the next request of the same size; a failed
// cudaMalloc releases the cached slabs of that device and retries, and
// sv_release_cached() returns everything to the driver.  Callers synchronise
// their stream before freeing (sv_destroy / svb_destroy), so a cached slab is
// idle when it is reused.
//
// Slabs exported over CUDA IPC (sv_ipc_handle / svb_ipc_handles) may still be
// mapped by peer processes after their owner freed them into the cache: CUDA
// leaves freeing an exported allocation before every importer closed it
// undefined.  Such slabs are marked and never returned to the driver -- neither
// by the out-of-memory retry nor by sv_release_cached -- until the distributed
// layer has closed every mapping on every rank and calls sv_ipc_unexport_all
// (distributed.release_peer_maps, after its barrier).  They can still be reused
// for the next same-size state of this process, which is what the peers' cached
// mappings rely on.
#include <mutex>
#include <unordered_set>
#include <vector>

#include "sv_common.cuh"
#include "sv_kernels.cuh"
#include "svb200.h"

namespace sv {

namespace {
struct Slab {
    int device;
    size_t bytes;
    void* ptr;
};
std::mutex& slab_mu() {
    static std::mutex* m = new std::mutex;
    return *m;
}
std::vector<Slab>& slabs() {
    static std::vector<Slab>* v = new std::vector<Slab>;
    return *v;
}
std::unordered_set<void*>& exported() {
    static std::unordered_set<void*>* s = new std::unordered_set<void*>;
    return *s;
}
constexpr size_t kMinCached = 1ull << 20;

void release_device(int device) {
    std::vector<Slab> drop;
    {
        std::lock_guard<std::mutex> lk(slab_mu());
        auto& v = slabs();
        const auto& ex = exported();
        for (size_t i = 0; i < v.size();) {
            if ((device < 0 || v[i].device == device) && !ex.count(v[i].ptr)) {
                drop.push_back(v[i]);
                v[i] = v.back();
                v.pop_back();
            } else {
                ++i;
            }
        }
    }
    int cur = 0;
    cudaGetDevice(&cur);
    for (const Slab& s : drop) {
        cudaSetDevice(s.device);
        cudaFree(s.ptr);
    }
    cudaSetDevice(cur);
}
}  // namespace

cudaError_t slab_alloc(void** p, size_t bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    {   // (slabs below kMinCached are only cached while exported)
        std::lock_guard<std::mutex> lk(slab_mu());
        auto& v = slabs();
        for (size_t i = 0; i < v.size(); ++i)
            if (v[i].device == dev && v[i].bytes == bytes) {
                *p = v[i].ptr;
                v[i] = v.back();
                v.pop_back();
                return cudaSuccess;
            }
    }
    cudaError_t e = cudaMalloc(p, bytes);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        release_device(dev);
        e = cudaMalloc(p, bytes);
    }
    return e;
}

void slab_free(void* p, size_t bytes) {
    if (!p) return;
    if (bytes < kMinCached) {
        {
            std::lock_guard<std::mutex> lk(slab_mu());
            if (exported().count(p)) {      // a peer may still map it: keep it (cached) until unexported
                int dev = 0;
                cudaGetDevice(&dev);
                slabs().push_back({dev, bytes, p});
                return;
            }
        }
        cudaFree(p);
        return;
    }
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(slab_mu());
    slabs().push_back({dev, bytes, p});
}

void slab_mark_exported(void* p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(slab_mu());
    exported().insert(p);
}

size_t slab_exported_count() {
    std::lock_guard<std::mutex> lk(slab_mu());
    return exported().size();
}

void slab_unexport_all() {
    std::lock_guard<std::mutex> lk(slab_mu());
    exported().clear();
}

size_t slab_cached_bytes() {
    std::lock_guard<std::mutex> lk(slab_mu());
    size_t t = 0;
    for (const Slab& s : slabs()) t += s.bytes;
    return t;
}

// Stream-ordered scratch (measurement partials, pair-dot rows, patch lists) comes from
// the device's default pool; with the default release threshold of 0 the pool hands
// its memory back at every synchronisation and the next cudaMallocAsync maps it
// again (~1-2 ms of host time).  Keep up to 256 MB of freed scratch in the pool.
void keep_scratch_pool(int device) {
    static bool done[64] = {false};
    if (device < 0 || device >= 64 || done[device]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = 256ull << 20;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done[device] = true;
}

}  // namespace sv

extern "C" {

int sv_release_cached(void) {
    sv::release_device(-1);
    return SV_OK;
}

int sv_cached_bytes(uint64_t* out) {
    *out = sv::slab_cached_bytes();
    return SV_OK;
}

int sv_ipc_unexport_all(uint64_t* was_exported) {
    if (was_exported) *was_exported = sv::slab_exported_count();
    sv::slab_unexport_all();
    return SV_OK;
}

}  // extern "C"
