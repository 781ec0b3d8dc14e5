// tokens.cuh -- parameters of the token-level merge kernel (tokens.cu).
#pragma once
#include <cstdint>

#include "common.cuh"

struct MergeParams {
    DevTables T;
    const uint32_t *tok;                // input tokens (internal ids), sequences back to back
    const unsigned long long *offs;     // [n_seqs + 1]
    unsigned long long n_seqs;
    uint32_t *arena;                    // ENGINE_BYTES(max length) per CTA, in words
    unsigned long long arena_words_per_cta;
    uint32_t *out;                      // sequence s -> out[offs[s] .. offs[s] + counts[s])
    unsigned long long *counts;         // [n_seqs]
    int strict;
    uint32_t n_ids;                     // ids the tables cover; a larger one fails its sequence
};

#ifdef __CUDACC__
cudaError_t launch_merge_tokens(const MergeParams &Q, int grid, cudaStream_t s);
#endif
