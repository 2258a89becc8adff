// Pinned host memory setup cost on the GPU box (the slow tier of sv_tier.cu):
//   nvcc -O2 -o tools/pin_probe tools/pin_probe.cu -lpthread && tools/pin_probe 16
// (a) cudaHostAlloc of 1 GiB blocks, serial; (b) the same from 8 threads;
// (c) mmap + MADV_HUGEPAGE + parallel first touch + cudaHostRegister per block.
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
    const int gib = argc > 1 ? atoi(argv[1]) : 16;
    const size_t blk = 1ull << 30;
    cudaFree(0);
    std::vector<void*> p(gib);
    double t = now();
    for (int i = 0; i < gib; ++i) cudaHostAlloc(&p[i], blk, cudaHostAllocPortable | cudaHostAllocMapped);
    printf("{\"serial_hostalloc_s\": %.3f, ", now() - t);
    for (void* q : p) cudaFreeHost(q);
    t = now();
    {
        std::vector<std::thread> th;
        for (int k = 0; k < 8; ++k)
            th.emplace_back([&, k] {
                for (int i = k; i < gib; i += 8) cudaHostAlloc(&p[i], blk, cudaHostAllocPortable | cudaHostAllocMapped);
            });
        for (auto& x : th) x.join();
    }
    printf("\"threads8_hostalloc_s\": %.3f, ", now() - t);
    for (void* q : p) cudaFreeHost(q);
    t = now();
    {
        std::vector<std::thread> th;
        for (int k = 0; k < 8; ++k)
            th.emplace_back([&, k] {
                for (int i = k; i < gib; i += 8) {
                    void* m = mmap(nullptr, blk, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
                    madvise(m, blk, MADV_HUGEPAGE);
                    memset(m, 0, blk);
                    p[i] = m;
                }
            });
        for (auto& x : th) x.join();
    }
    const double touch = now() - t;
    double t2 = now();
    {
        std::vector<std::thread> th;
        for (int k = 0; k < 8; ++k)
            th.emplace_back([&, k] {
                for (int i = k; i < gib; i += 8) cudaHostRegister(p[i], blk, cudaHostRegisterPortable | cudaHostRegisterMapped);
            });
        for (auto& x : th) x.join();
    }
    printf("\"mmap_huge_touch_s\": %.3f, \"register8_s\": %.3f, \"err\": \"%s\", \"gib\": %d}\n", touch, now() - t2,
           cudaGetErrorString(cudaGetLastError()), gib);
    return 0;
}
