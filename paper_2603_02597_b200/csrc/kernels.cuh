// kernels.cuh -- the fused encode kernel and its launch parameters.
//
// k_encode is ONE persistent launch per batch.  Each CTA repeatedly takes the
// next TILE bytes (dynamic tile counter, so tiles are taken in order) and:
//   1. stages the tile (+HALO) in shared memory, maps bytes to ids,
//   2. marks segment boundaries: junction bitmap misses, document starts,
//      fixed-offset chunk cuts (P-default semantics),
//   3. encodes every segment that STARTS in the tile:
//        len 1                    base id
//        2..32, vocab string      one memo probe
//        2..32, other             one warp, exact multi-merge in registers
//        33..MED_MAX              whole CTA, exact multi-merge in scratch
//        longer ("giant")         whole CTA, exact multi-merge in the arena
//   4. publishes its id count and finds its output offset by decoupled
//      look-back over the tile status words,
//   5. stores ids (coalesced) and the CSR offsets of documents starting in it.
#pragma once
#include "common.cuh"
#include "engine.cuh"
#include "warp_engine.cuh"

#define TILE 2048            // bytes per tile
#define HALO 256             // bytes staged past the tile end
#define LD (TILE + HALO)     // bytes staged per tile
#define NT 256               // threads per CTA
#define SHORT_MAX 32         // longest segment a warp encodes in registers
#define MED_MAX LD           // longest segment encoded in per-CTA scratch
#define NOSEG 0xFFFFu        // segment end lies past the staged bytes

// Per-call device state, zeroed at the start of every encode.
struct EncodeState {
    unsigned long long tile_counter;
    unsigned long long arena_used;  // u32 words requested from the arena
    unsigned long long overflow;
    unsigned long long error;
    // counters
    unsigned long long n_ids;
    unsigned long long n_segments;
    unsigned long long memo_hits;
    unsigned long long short_merges;
    unsigned long long medium_segments;
    unsigned long long giant_segments;
    unsigned long long giant_bytes;
    unsigned long long engine_passes;
};

struct EncodeParams {
    DevTables T;
    const uint8_t *bytes;
    unsigned long long n_bytes;
    const long long *doc_offs;
    unsigned long long n_docs;
    unsigned long long max_seq_len, chunk_budget;
    uint32_t *out_ids;
    long long *out_offs;
    EncodeState *st;       // this call's state (zeroed by the previous call)
    EncodeState *st_next;  // the next call's state, zeroed here by CTA 0
    unsigned long long *status;  // [n_tiles] look-back words
    uint8_t *med_scratch;        // [grid * MED_BYTES]
    uint8_t *arena;              // giant segments
    unsigned long long arena_cap;
    unsigned long long n_tiles;
    unsigned int epoch;          // look-back tag (20 bits)
    int strict;
};

// engine scratch for n tokens: tok, tok2 (u32) + pr, pr2 (uint2) + sel (u8)
#define ENGINE_BYTES(n) ((size_t)(n) * 25 + 64)
#define MED_BYTES ENGINE_BYTES(MED_MAX)
