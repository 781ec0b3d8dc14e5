// Overlap probe: a 148 x 1024 kernel (cooperative or not, on the legacy
// stream or a created one) whose CTAs wait for per-piece arrival words that a
// non-blocking copy stream DMAs after each piece -- the shape of the
// overlapped host encode.  Prints when each piece's word was seen (globaltimer,
// relative to the kernel's first CTA) and the host wall time of the whole call.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/bin/overlap_probe tools/overlap_probe.cu
#include <chrono>
#include <algorithm>
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void k_wait(const unsigned *arrive, unsigned tag, int pieces, unsigned long long *stamps) {
    extern __shared__ unsigned char sm[];
    if (threadIdx.x == 0) {
        const unsigned long long t0 = gt();
        atomicMin(&stamps[0], t0);
        const int k = blockIdx.x % pieces;  // CTA c waits for piece c % pieces
        while (*(volatile const unsigned *)&arrive[32 * k] != tag) __nanosleep(256);
        atomicMax(&stamps[1 + k], gt());
        sm[0] = 1;
    }
    __syncthreads();
}

int main() {
    const int pieces = 4;
    const size_t piece = 192 << 10;
    unsigned *d_arrive, *h_tag;
    unsigned long long *d_st, h_st[8];
    (void)h_st;
    char *h_pin, *d_buf;
    cudaMalloc(&d_arrive, 32 * 32 * 4);
    cudaMemset(d_arrive, 0, 32 * 32 * 4);
    cudaHostAlloc((void **)&h_tag, 64, 0);
    cudaHostAlloc((void **)&h_pin, pieces * piece, cudaHostAllocMapped);
    cudaMalloc(&d_buf, pieces * piece);
    cudaMalloc(&d_st, 64);
    cudaStream_t s_copy, s_mine;
    cudaStreamCreateWithFlags(&s_copy, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s_mine, cudaStreamNonBlocking);
    cudaFuncSetAttribute(k_wait, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10);
    unsigned tag = 0;
    typedef CUresult (*WriteValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
    WriteValue32 wv = nullptr;
    cudaDriverEntryPointQueryResult qr;
    cudaGetDriverEntryPoint("cuStreamWriteValue32", (void **)&wv, cudaEnableDefault, &qr);
    printf("cuStreamWriteValue32 %s\n", wv ? "found" : "missing");
    for (int variant = 0; variant < 8; ++variant) {
        const int coop = 1;
        cudaStream_t s = 0;
        const int np = variant < 2 ? 1 : variant < 4 ? 2 : variant < 6 ? 4 : 8;
        const int use_wv = variant & 1;
        if (use_wv && !wv) continue;
        const size_t pc = pieces * piece / np;
        double best = 1e9;
        unsigned long long last[16] = {};
        for (int it = 0; it < 20; ++it) {
            cudaMemsetAsync(d_st, 0, 64, s);
            unsigned long long init = ~0ull;
            cudaMemcpyAsync(d_st, &init, 8, cudaMemcpyHostToDevice, s);
            cudaStreamSynchronize(s);
            *h_tag = ++tag;
            auto t0 = std::chrono::steady_clock::now();
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(148);
            cfg.blockDim = dim3(1024);
            cfg.dynamicSmemBytes = 200 << 10;
            cfg.stream = s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeCooperative;
            at[0].val.cooperative = 1;
            cfg.attrs = at;
            cfg.numAttrs = coop;
            cudaLaunchKernelEx(&cfg, k_wait, (const unsigned *)d_arrive, tag, np, d_st);
            for (int k = 0; k < np; ++k) {
                cudaMemcpyAsync(d_buf + k * pc, h_pin + k * pc, pc, cudaMemcpyHostToDevice, s_copy);
                if (use_wv) wv((CUstream)s_copy, (CUdeviceptr)(d_arrive + 32 * k), tag, 0);
                else cudaMemcpyAsync(d_arrive + 32 * k, h_tag, 4, cudaMemcpyHostToDevice, s_copy);
            }
            cudaStreamSynchronize(s);
            auto t1 = std::chrono::steady_clock::now();
            const double us = std::chrono::duration<double, std::micro>(t1 - t0).count();
            cudaMemcpy(h_st, d_st, 64, cudaMemcpyDeviceToHost);
            if (us < best) {
                best = us;
                for (int k = 0; k < 8; ++k) last[k] = h_st[k];
            }
        }
        printf("%d pieces of %zu KB, flags by %s: host %.1f us; piece seen at", np, pc >> 10,
               use_wv ? "cuStreamWriteValue32" : "4-byte H2D copy", best);
        for (int k = 0; k < np && k < 7; ++k) printf(" %.1f", (last[1 + k] - last[0]) / 1e3);
        printf(" us after the first CTA\n");
    }
    {  // the input split over 1..4 copy streams (one piece + arrival word each), kernel waiting
        cudaStream_t cs[4];
        for (auto &c : cs) cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking);
        for (int ns = 1; ns <= 4; ns *= 2) {
            const size_t pc = pieces * piece / ns;
            double best = 1e9;
            unsigned long long last[8] = {};
            for (int it = 0; it < 20; ++it) {
                cudaMemsetAsync(d_st, 0, 64, 0);
                unsigned long long init = ~0ull;
                cudaMemcpyAsync(d_st, &init, 8, cudaMemcpyHostToDevice, 0);
                cudaStreamSynchronize(0);
                *h_tag = ++tag;
                auto t0 = std::chrono::steady_clock::now();
                for (int k = 0; k < ns; ++k) {
                    cudaMemcpyAsync(d_buf + k * pc, h_pin + k * pc, pc, cudaMemcpyHostToDevice, cs[k]);
                    cudaMemcpyAsync(d_arrive + 32 * k, h_tag, 4, cudaMemcpyHostToDevice, cs[k]);
                }
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(148);
                cfg.blockDim = dim3(1024);
                cfg.dynamicSmemBytes = 200 << 10;
                cfg.stream = 0;
                cudaLaunchKernelEx(&cfg, k_wait, (const unsigned *)d_arrive, tag, ns, d_st);
                cudaStreamSynchronize(0);
                auto t1 = std::chrono::steady_clock::now();
                const double us = std::chrono::duration<double, std::micro>(t1 - t0).count();
                cudaMemcpy(h_st, d_st, 64, cudaMemcpyDeviceToHost);
                if (us < best) {
                    best = us;
                    for (int k = 0; k < 8; ++k) last[k] = h_st[k];
                }
            }
            printf("%d copy streams x %zu KB (DMA first, then the kernel): host %.1f us; seen at", ns, pc >> 10, best);
            for (int k = 0; k < ns; ++k) printf(" %.1f", (last[1 + k] - last[0]) / 1e3);
            printf(" us after the first CTA\n");
        }
    }
    {  // plain H2D of the whole buffer, timed alone
        double best = 1e9;
        for (int it = 0; it < 20; ++it) {
            auto t0 = std::chrono::steady_clock::now();
            cudaMemcpyAsync(d_buf, h_pin, pieces * piece, cudaMemcpyHostToDevice, s_copy);
            cudaStreamSynchronize(s_copy);
            auto t1 = std::chrono::steady_clock::now();
            best = std::min(best, std::chrono::duration<double, std::micro>(t1 - t0).count());
        }
        printf("one H2D of %zu KB alone: %.1f us\n", pieces * piece >> 10, best);
    }
    cudaError_t e = cudaGetLastError();
    printf("last error: %s\n", cudaGetErrorString(e));
    return 0;
}
