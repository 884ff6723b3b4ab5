// register_probe.cu -- can a pageable caller's array be DMA'd in place? Parallel
// cudaHostRegister / cudaHostUnregister throughput of 64 MB page-aligned pieces with T threads,
// and the H2D rate from the registered pieces.  nvcc -O2 -o register_probe register_probe.cu
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
    const size_t bytes = size_t(16) << 30, piece = size_t(64) << 20;
    char* host = static_cast<char*>(std::aligned_alloc(4096, bytes));
    std::memset(host, 1, bytes);  // resident pages, like a filled std::vector
    char* dev = nullptr;
    cudaMalloc(&dev, bytes);
    const size_t np = bytes / piece;
    for (int nt : {1, 4, 8, 16}) {
        double t0 = now();
        std::vector<std::thread> th;
        for (int t = 0; t < nt; ++t)
            th.emplace_back([&, t] {
                for (size_t p = t; p < np; p += nt) cudaHostRegister(host + p * piece, piece, 0);
            });
        for (auto& x : th) x.join();
        double t1 = now();
        cudaMemcpy(dev, host, bytes, cudaMemcpyHostToDevice);
        double t2 = now();
        th.clear();
        for (int t = 0; t < nt; ++t)
            th.emplace_back([&, t] {
                for (size_t p = t; p < np; p += nt) cudaHostUnregister(host + p * piece);
            });
        for (auto& x : th) x.join();
        double t3 = now();
        std::printf("%2d threads: register %.1f GB/s, H2D from registered %.1f GB/s, unregister %.1f GB/s\n",
                    nt, bytes / (t1 - t0) / 1e9, bytes / (t2 - t1) / 1e9, bytes / (t3 - t2) / 1e9);
    }
    return 0;
}
