// kernels.cuh -- the encode kernels and their launch parameters.
//
//   K0 k_windows  one thread per WIN-byte window: owning document (binary
//                 search of the doc offsets), and whether the window holds no
//                 segment boundary at all ("clear").  A segment containing a
//                 clear window is "giant"; every other segment is < 2*WIN bytes.
//   K1 k_giant    finds runs of clear windows (= giant segments), resolves
//                 their exact extent and runs the CTA engine on each in a
//                 global-memory arena.
//   K2 k_tile     persistent, one TILE of bytes per iteration: byte -> id map,
//                 junction/document/chunk boundaries, per-segment BPE (memo
//                 probe, per-thread greedy, CTA engine for medium segments),
//                 decoupled look-back for the output offset, coalesced id
//                 store, document offsets.
#pragma once
#include <cuda/atomic>

#include "common.cuh"
#include "engine.cuh"

#define TILE 2048            // bytes per tile
#define WIN 1024             // giant-detection window (TILE % WIN == 0)
#define HALO 256             // bytes loaded past the tile end
#define LD (TILE + HALO)     // bytes held in shared memory per tile
#define NT 256               // threads per CTA (all kernels)
#define SHORT_MAX 32         // longest segment merged by one thread
#define MED_MAX (2 * WIN)    // longest non-giant segment (+1)
#define NOSEG 0xFFFFu        // "segment end beyond the loaded bytes"
#define PENDING 0xFFFFFFFFu  // count filled by the cooperative phase

// Per-call device state, zeroed by k_windows.
struct EncodeState {
    unsigned long long tile_counter;
    unsigned long long n_giant;
    unsigned long long arena_used;
    unsigned long long overflow;
    unsigned long long error;
    // stats
    unsigned long long n_ids;
    unsigned long long n_segments;
    unsigned long long memo_hits;
    unsigned long long short_merges;
    unsigned long long medium_segments;
    unsigned long long giant_segments;
    unsigned long long giant_bytes;
    unsigned long long engine_passes;
};

struct GiantRec {
    unsigned long long start, end;  // byte positions [start, end)
    unsigned long long out_off;     // element offset of the result in the arena (u32 units)
    unsigned long long count;       // ids produced
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
    // workspace
    EncodeState *st;
    long long *window_doc;       // [n_win]
    uint8_t *wclear;             // [n_win]
    int *giant_at;               // [n_win] record index of the giant segment starting in window
    GiantRec *recs;              // [n_win]
    unsigned long long *status;  // [n_tiles] look-back words
    uint8_t *med_scratch;        // [grid_tile * MED_BYTES]
    uint8_t *arena;
    unsigned long long arena_cap;
    unsigned long long n_win, n_tiles;
    unsigned int epoch;  // look-back tag (20 bits)
    int strict;
};

#define MED_BYTES ((size_t)MED_MAX * 25 + 64)
