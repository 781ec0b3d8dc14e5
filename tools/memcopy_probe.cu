// Host copy / PCIe bandwidth probe (build: nvcc -O2 -o tools/bin/memcopy_probe tools/memcopy_probe.cu).
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
#include <cstdlib>
#include <cuda_runtime.h>
int main() {
    size_t n = 256ull << 20;
    char *a = (char*)malloc(n), *b = (char*)malloc(n);
    memset(a, 1, n); memset(b, 2, n);
    char *p; cudaHostAlloc((void**)&p, n, cudaHostAllocMapped);
    memset(p, 0, n);
    for (int T : {1, 2, 4, 8, 12, 16, 24, 32}) {
        for (int rep = 0; rep < 2; ++rep) {
            auto t0 = std::chrono::steady_clock::now();
            std::vector<std::thread> th;
            size_t ch = n / T;
            for (int i = 0; i < T; ++i) th.emplace_back([=]{ memcpy(p + i*ch, a + i*ch, ch); });
            for (auto &t : th) t.join();
            double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            if (rep) printf("T=%d pageable->pinned %.1f GB/s\n", T, n / s / 1e9);
        }
    }
    for (int T : {8, 16}) {
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        size_t ch = n / T;
        for (int i = 0; i < T; ++i) th.emplace_back([=]{ memcpy(b + i*ch, p + i*ch, ch); });
        for (auto &t : th) t.join();
        double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        printf("T=%d pinned->pageable %.1f GB/s\n", T, n / s / 1e9);
    }
    auto t0 = std::chrono::steady_clock::now();
    cudaHostRegister(b, n, 0);
    double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    printf("cudaHostRegister 256MB %.2f ms\n", s*1e3);
    t0 = std::chrono::steady_clock::now();
    cudaHostUnregister(b);
    s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    printf("cudaHostUnregister 256MB %.2f ms\n", s*1e3);
    char *d; cudaMalloc(&d, n);
    for (int rep = 0; rep < 3; ++rep) {
        t0 = std::chrono::steady_clock::now();
        cudaMemcpy(d, a, n, cudaMemcpyHostToDevice);
        s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        printf("pageable H2D %.1f GB/s\n", n / s / 1e9);
    }
    for (int rep = 0; rep < 2; ++rep) {
        t0 = std::chrono::steady_clock::now();
        cudaMemcpy(d, p, n, cudaMemcpyHostToDevice);
        s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        printf("pinned H2D %.1f GB/s\n", n / s / 1e9);
        t0 = std::chrono::steady_clock::now();
        cudaMemcpy(p, d, n, cudaMemcpyDeviceToHost);
        s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        printf("pinned D2H %.1f GB/s\n", n / s / 1e9);
    }
    // both directions at once (two streams, pinned buffers): the ceiling of a
    // streamed encode that reads bytes in and writes ids out
    char *p2; cudaHostAlloc((void**)&p2, n, cudaHostAllocMapped);
    char *d2; cudaMalloc(&d2, n);
    cudaStream_t s1, s2; cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    for (int rep = 0; rep < 3; ++rep) {
        cudaDeviceSynchronize();
        t0 = std::chrono::steady_clock::now();
        cudaMemcpyAsync(d, p, n, cudaMemcpyHostToDevice, s1);
        cudaMemcpyAsync(p2, d2, n, cudaMemcpyDeviceToHost, s2);
        cudaDeviceSynchronize();
        s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        printf("pinned H2D + D2H concurrently: %.1f GB/s each way, %.1f GB/s total\n", n / s / 1e9, 2 * n / s / 1e9);
    }
}
