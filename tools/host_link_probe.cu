// host_link_probe.cu -- what a pageable caller's data can move at on this host:
// parallel memcpy pageable -> page-locked with 1..16 threads, cudaHostRegister of a pageable
// block, and H2D from page-locked / pageable memory.  nvcc -O2 -o host_link_probe host_link_probe.cu
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
    const size_t bytes = size_t(4) << 30;
    std::vector<char> pageable(bytes, 1);  // touched: resident pages, like a filled std::vector
    char* pinned = nullptr;
    cudaMallocHost(&pinned, bytes);
    std::memset(pinned, 0, bytes);
    void* dev = nullptr;
    cudaMalloc(&dev, bytes);
    for (int nt : {1, 2, 4, 8, 12, 16}) {
        double best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
            const double t0 = now();
            std::vector<std::thread> th;
            const size_t piece = bytes / nt;
            for (int t = 0; t < nt; ++t)
                th.emplace_back([&, t] { std::memcpy(pinned + t * piece, pageable.data() + t * piece, piece); });
            for (auto& x : th) x.join();
            best = std::min(best, now() - t0);
        }
        std::printf("memcpy pageable->pinned %2d threads: %.1f GB/s\n", nt, bytes / best / 1e9);
    }
    {
        const double t0 = now();
        cudaError_t e = cudaHostRegister(pageable.data(), bytes, cudaHostRegisterDefault);
        const double t1 = now();
        std::printf("cudaHostRegister 4 GiB: %.3f s (%.1f GB/s) %s\n", t1 - t0, bytes / (t1 - t0) / 1e9,
                    cudaGetErrorString(e));
        const double t2 = now();
        cudaMemcpy(dev, pageable.data(), bytes, cudaMemcpyHostToDevice);
        const double t3 = now();
        std::printf("H2D from registered: %.1f GB/s\n", bytes / (t3 - t2) / 1e9);
        const double t4 = now();
        cudaHostUnregister(pageable.data());
        std::printf("cudaHostUnregister: %.3f s\n", now() - t4);
    }
    for (int k = 0; k < 2; ++k) {
        const double t0 = now();
        cudaMemcpy(dev, pinned, bytes, cudaMemcpyHostToDevice);
        const double t1 = now();
        cudaMemcpy(dev, pageable.data(), bytes, cudaMemcpyHostToDevice);
        const double t2 = now();
        std::printf("H2D pinned %.1f GB/s, pageable (driver staging) %.1f GB/s\n", bytes / (t1 - t0) / 1e9,
                    bytes / (t2 - t1) / 1e9);
    }
    return 0;
}
