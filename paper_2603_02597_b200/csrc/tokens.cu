// tokens.cu -- token-level merges on the device: the reference's engine entry
// points sequential_bpe (engines.py:269-335) and run_block_engine
// (engines.py:338-403) take token ids, not bytes.  One CTA per sequence runs
// the exact CTA engine (engine.cuh: strict one-merge passes when the table is
// not well-formed, exact multi-merge passes otherwise) in its own slice of the
// arena; the result is compacted in place of the input.  Tokens that no rule
// mentions are split off by the host (they can never merge).
#include <cuda_runtime.h>

#include <algorithm>

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
            bad |= t > Q.n_ids;
            M.tok[j] = t;
        }
        if (__syncthreads_or(bad)) {  // an id the tables do not cover: reported, not merged
            if (threadIdx.x == 0) Q.counts[s] = ~0ull;
            continue;
        }
        uint32_t passes = 0;
        const uint32_t *res = M.tok;
        const EngineExt ext{Q.trace ? Q.trace + lo : nullptr, (long long)s == Q.fault_seq};
        const uint32_t cnt =
            n ? engine_run_g<BlockGroup, true>(Q.T, M, (uint32_t)n, Q.strict != 0, g, &passes, &res, ext) : 0u;
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

// ---------------------------------------------------------------- lane-engine steps
//
// The reference's lane engine (engines.py:107-217) is a CPU model of one pass
// of the paper's kernel: eval_pairs (probe every adjacent pair, reduce to the
// lowest (rank, position)), and the two one-merge compactions.  These kernels
// are those steps on the device, callable one at a time like the reference's
// functions (the batch path never uses them: k_encode fuses everything).

// eval_pairs (engines.py:133-168): one CTA strides over the pairs; out[0] =
// position (~0 when no pair is in the table), out[1] = rank, out[2] = new id.
__global__ void __launch_bounds__(1024) k_eval_pairs(const DevTables T, const uint32_t *tok, unsigned long long n,
                                                     unsigned long long *out) {
    __shared__ EngineShared sh;
    unsigned long long best = ~0ull;
    for (unsigned long long i = threadIdx.x; i + 1 < n; i += blockDim.x) {
        const PairHit h = probe_pair(T, tok[i], tok[i + 1]);
        if (h.rank != GPUBPE_INF) {
            const unsigned long long k = ((unsigned long long)h.rank << 32) | i;
            best = k < best ? k : best;
        }
    }
    best = block_min_u64(best, sh);
    if (threadIdx.x == 0) {
        if (best == ~0ull) {
            out[0] = ~0ull;
        } else {
            const uint32_t pos = (uint32_t)best;
            const PairHit h = probe_pair(T, tok[pos], tok[pos + 1]);
            out[0] = pos;
            out[1] = h.rank;
            out[2] = out_id(T, h.nw);
        }
    }
}

// compact_double_buffer (engines.py:197-217): every source index maps to its
// destination directly -- no scan, no ordering between writes.
__global__ void k_compact_direct(const uint32_t *tok, unsigned long long n, unsigned long long best,
                                 uint32_t nw, uint32_t *out) {
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i + 1 < n;
         i += (unsigned long long)gridDim.x * blockDim.x)
        out[i] = i < best ? tok[i] : (i == best ? nw : tok[i + 1]);
}

// compact_scan (engines.py:171-194): removal flags, exclusive prefix sum of
// the flags (one CTA, chunk by chunk with a carry), scatter of the kept
// tokens to index - removed_before; the merged slot takes the new token.
__global__ void __launch_bounds__(1024) k_compact_scan(const uint32_t *tok, unsigned long long n,
                                                       unsigned long long best, uint32_t nw, uint32_t *out) {
    __shared__ EngineShared sh;
    unsigned long long carry = 0;
    for (unsigned long long b = 0; b < n; b += blockDim.x) {
        const unsigned long long j = b + threadIdx.x;
        const uint32_t remove = j < n && j == best + 1;
        uint32_t total;
        const unsigned long long before = carry + block_excl_sum(remove, sh, &total);
        if (j < n && !remove) out[j - before] = j == best ? nw : tok[j];
        carry += total;
    }
}

// PackedPairTable.lookup_keys_into (merge_table.py:170-230): packed keys
// (left << 32) | right -> hit flag and the packed value (new << 32) | rank;
// the empty-slot sentinel key is always a miss (merge_table.py:211-214).
__global__ void k_lookup_keys(const DevTables T, const unsigned long long *keys, unsigned long long m,
                              uint8_t *hit, unsigned long long *vals) {
    const unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const unsigned long long k = keys[i];
    PairHit h{GPUBPE_INF, 0};
    if (k != ~0ull) h = probe_pair(T, (uint32_t)(k >> 32), (uint32_t)k);
    hit[i] = h.rank != GPUBPE_INF;
    vals[i] = h.rank != GPUBPE_INF ? ((unsigned long long)out_id(T, h.nw) << 32) | h.rank : 0ull;
}

cudaError_t launch_eval_pairs(const DevTables &T, const uint32_t *tok, unsigned long long n,
                              unsigned long long *out, cudaStream_t s) {
    k_eval_pairs<<<1, 1024, 0, s>>>(T, tok, n, out);
    return cudaGetLastError();
}

cudaError_t launch_compact(const uint32_t *tok, unsigned long long n, unsigned long long best, uint32_t nw,
                           uint32_t *out, int scan, cudaStream_t s) {
    if (n < 2) return cudaSuccess;
    if (scan)
        k_compact_scan<<<1, 1024, 0, s>>>(tok, n, best, nw, out);
    else
        k_compact_direct<<<(unsigned int)std::min<unsigned long long>((n + 255) / 256, 148ull * 8), 256, 0, s>>>(
            tok, n, best, nw, out);
    return cudaGetLastError();
}

cudaError_t launch_lookup_keys(const DevTables &T, const unsigned long long *keys, unsigned long long m,
                               uint8_t *hit, unsigned long long *vals, cudaStream_t s) {
    if (m == 0) return cudaSuccess;
    k_lookup_keys<<<(unsigned int)((m + 255) / 256), 256, 0, s>>>(T, keys, m, hit, vals);
    return cudaGetLastError();
}
