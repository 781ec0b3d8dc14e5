// Launch-overhead probe: event-timed empty kernels in the k_encode launch
// configuration (148 x 1024 threads, ~200 KB dynamic smem), cooperative or not.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/bin/launch_probe tools/launch_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_empty(int *p) { if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] = 1; }
__global__ void k_sync(int *ctr, int n) {  // one grid barrier
    __syncthreads();
    if (threadIdx.x == 0) {
        atomicAdd(ctr, 1);
        while (atomicAdd(ctr, 0) < n) {}
    }
    __syncthreads();
}
#include <chrono>
static double host_us(void (*f)(), int k) {
    for (int i = 0; i < 10; ++i) f();
    cudaDeviceSynchronize();
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < k; ++i) f();
    auto t1 = std::chrono::steady_clock::now();
    cudaDeviceSynchronize();
    return std::chrono::duration<double, std::micro>(t1 - t0).count() / k;
}
static int g_coop = 0, g_smem = 0;
static void launch_one() {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148); cfg.blockDim = dim3(1024); cfg.dynamicSmemBytes = g_smem;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeCooperative; at[0].val.cooperative = 1;
    cfg.attrs = at; cfg.numAttrs = g_coop;
    cudaLaunchKernelEx(&cfg, k_empty, (int *)nullptr);
}
static char *g_h, *g_d;
static void memcpy_one() { cudaMemcpyAsync(g_d, g_h, 4096, cudaMemcpyHostToDevice, 0); }
static cudaEvent_t g_ev;
static void event_one() { cudaEventRecord(g_ev, 0); }
static void attr_one() { cudaPointerAttributes pa; cudaPointerGetAttributes(&pa, g_h); }

int main() {
    cudaMallocHost(&g_h, 1 << 20); cudaMalloc(&g_d, 1 << 20); cudaEventCreate(&g_ev);
    for (int smem : {0, 200 * 1024}) {
        cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        for (int coop : {0, 1}) {
            g_coop = coop; g_smem = smem;
            printf("host enqueue: launch smem %6d coop %d  %.2f us\n", smem, coop, host_us(launch_one, 200));
        }
    }
    printf("host enqueue: cudaMemcpyAsync 4 KB pinned H2D %.2f us\n", host_us(memcpy_one, 200));
    printf("host enqueue: cudaEventRecord %.2f us\n", host_us(event_one, 200));
    printf("host: cudaPointerGetAttributes %.2f us\n", host_us(attr_one, 200));

    int *ctr; cudaMalloc(&ctr, 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int smem : {0, 200 * 1024}) {
        cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_sync, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        for (int coop : {0, 1}) {
            for (int which : {0, 1}) {
                float best = 1e9, sum = 0;
                for (int it = 0; it < 50; ++it) {
                    cudaMemset(ctr, 0, 4);
                    cudaLaunchConfig_t cfg = {};
                    cfg.gridDim = dim3(148); cfg.blockDim = dim3(1024); cfg.dynamicSmemBytes = smem;
                    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeCooperative; at[0].val.cooperative = 1;
                    cfg.attrs = at; cfg.numAttrs = coop;
                    cudaEventRecord(a);
                    if (which == 0) cudaLaunchKernelEx(&cfg, k_empty, (int *)nullptr);
                    else cudaLaunchKernelEx(&cfg, k_sync, ctr, 148);
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    float ms; cudaEventElapsedTime(&ms, a, b);
                    if (it >= 5) { best = ms < best ? ms : best; sum += ms; }
                }
                printf("smem %6d coop %d %-8s min %.2f us  mean %.2f us  (%s)\n", smem, coop, which ? "barrier" : "empty",
                       best * 1e3, sum / 45 * 1e3, cudaGetErrorString(cudaGetLastError()));
            }
        }
    }
}
