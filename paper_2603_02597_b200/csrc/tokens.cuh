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
    uint32_t n_ids;                     // ids the tables cover (id n_ids itself: the inert
                                        // sentinel no rule mentions); a larger one fails its sequence
    unsigned long long *trace;          // nullable: sequence s's merges at trace[offs[s] ..]
                                        // as (pass << 32) | rank (engine.cuh EngineExt)
    long long fault_seq;                // sequence whose run takes the compaction fault, or -1
};

#ifdef __CUDACC__
cudaError_t launch_merge_tokens(const MergeParams &Q, int grid, cudaStream_t s);
#endif

#ifdef __CUDACC__
cudaError_t launch_eval_pairs(const DevTables &T, const uint32_t *tok, unsigned long long n,
                              unsigned long long *out, cudaStream_t s);
cudaError_t launch_compact(const uint32_t *tok, unsigned long long n, unsigned long long best, uint32_t nw,
                           uint32_t *out, int scan, cudaStream_t s);
cudaError_t launch_lookup_keys(const DevTables &T, const unsigned long long *keys, unsigned long long m,
                               uint8_t *hit, unsigned long long *vals, cudaStream_t s);
#endif
