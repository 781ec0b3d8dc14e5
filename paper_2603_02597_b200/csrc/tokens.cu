// tokens.cu -- token-level merges on the device: the reference's engine entry
// points sequential_bpe (engines.py:269-335) and run_block_engine
// (engines.py:338-403) take token ids, not bytes.  One CTA per sequence runs
// the exact CTA engine (engine.cuh: strict one-merge passes when the table is
// not well-formed, exact multi-merge passes otherwise) in its own slice of the
// arena; the result is compacted in place of the input.  Tokens that no rule
// mentions are split off by the host (they can never merge).
#include <cuda_runtime.h>

#include "../../include/gpubpe.h"
#include "common.cuh"
#include "engine.cuh"
#include "kernels.cuh"
#include "tokens.cuh"

__global__ void __launch_bounds__(1024) k_merge_tokens(const __grid_constant__ MergeParams Q) {
    __shared__ EngineShared sh;
    BlockGroup g{sh};
    uint32_t *mem = Q.arena + (unsigned long long)blockIdx.x * Q.arena_words_per_cta;
    for (unsigned long long s = blockIdx.x; s < Q.n_seqs; s += gridDim.x) {
        const unsigned long long lo = Q.offs[s], n = Q.offs[s + 1] - lo;
        EngineMem M;
        M.tok = mem;
        M.tok2 = M.tok + n;
        M.pr = reinterpret_cast<uint2 *>(M.tok2 + n);
        M.pr2 = M.pr + n;
        M.sel = reinterpret_cast<uint8_t *>(M.pr2 + n);
        int bad = 0;
        for (unsigned long long j = threadIdx.x; j < n; j += blockDim.x) {
            const uint32_t t = Q.tok[lo + j];
            bad |= t >= Q.n_ids;
            M.tok[j] = t;
        }
        if (__syncthreads_or(bad)) {  // an id the tables do not cover: reported, not merged
            if (threadIdx.x == 0) Q.counts[s] = ~0ull;
            continue;
        }
        uint32_t passes = 0;
        const uint32_t *res = M.tok;
        const uint32_t cnt = n ? engine_run_g(Q.T, M, (uint32_t)n, Q.strict != 0, g, &passes, &res) : 0u;
        for (uint32_t j = threadIdx.x; j < cnt; j += blockDim.x) Q.out[lo + j] = res[j];
        if (threadIdx.x == 0) Q.counts[s] = cnt;
        __syncthreads();
    }
}

cudaError_t launch_merge_tokens(const MergeParams &Q, int grid, cudaStream_t s) {
    if (Q.n_seqs == 0) return cudaSuccess;
    k_merge_tokens<<<grid, 1024, 0, s>>>(Q);
    return cudaGetLastError();
}
