// bounce_probe.cu -- pageable -> device upload through a ring of page-locked bounce blocks
// (DESIGN.md 3b): end-to-end GB/s for block sizes 1 MB .. 256 MB, T copy threads each owning a
// ring of K blocks and its own stream.   nvcc -O2 -o bounce_probe bounce_probe.cu -lpthread
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
    const size_t bytes = size_t(8) << 30;
    std::vector<char> pageable(bytes, 1);
    char* dev = nullptr;
    cudaMalloc(&dev, bytes);
    for (size_t blk : {size_t(1) << 20, size_t(4) << 20, size_t(16) << 20, size_t(64) << 20}) {
        for (int nt : {4, 8, 16}) {
            const int K = 3;
            std::vector<char*> ring(size_t(nt) * K);
            for (auto& r : ring) cudaMallocHost(&r, blk);
            std::vector<cudaStream_t> st(nt);
            std::vector<cudaEvent_t> ev(size_t(nt) * K);
            for (auto& s : st) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
            for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
            double best = 1e9;
            for (int rep = 0; rep < 2; ++rep) {
                cudaDeviceSynchronize();
                const double t0 = now();
                std::vector<std::thread> th;
                for (int t = 0; t < nt; ++t)
                    th.emplace_back([&, t] {
                        const size_t per = bytes / nt;
                        int n = 0;
                        for (size_t o = size_t(t) * per; o < size_t(t + 1) * per; o += blk, ++n) {
                            const int j = n % K;
                            char* b = ring[size_t(t) * K + j];
                            if (n >= K) cudaEventSynchronize(ev[size_t(t) * K + j]);
                            const size_t len = std::min(blk, size_t(t + 1) * per - o);
                            std::memcpy(b, pageable.data() + o, len);
                            cudaMemcpyAsync(dev + o, b, len, cudaMemcpyHostToDevice, st[t]);
                            cudaEventRecord(ev[size_t(t) * K + j], st[t]);
                        }
                        cudaStreamSynchronize(st[t]);
                    });
                for (auto& x : th) x.join();
                best = std::min(best, now() - t0);
            }
            std::printf("block %4zu MB, %2d threads x %d blocks: %.1f GB/s\n", blk >> 20, nt, K,
                        bytes / best / 1e9);
            for (auto& r : ring) cudaFreeHost(r);
            for (auto& s : st) cudaStreamDestroy(s);
            for (auto& e : ev) cudaEventDestroy(e);
        }
    }
    return 0;
}
