// kernels.cuh -- the fused encode kernel and its launch parameters.
//
// k_encode is ONE cooperative persistent launch per batch (grid = one CTA of
// NW warps per SM).  The input is processed in ROUNDS of up to R tiles of WT
// bytes; each round has two phases separated by one grid barrier.
//
// Phase A (encode; every WARP autonomous, no waiting): a warp takes the next
// tile of the round from a counter and
//   1. stages the tile (+HALO) in its own shared memory (16-B loads),
//   2. marks cut positions: junction-bitmap misses (bitmap in smem), document
//      starts, fixed-offset chunk cuts (P-default semantics), end of input,
//   3. encodes every segment that STARTS in the tile, lane L owning the
//      segments that start in bytes [16L, 16L+16):
//        len 1               base id
//        2..SHORT_MAX        one memo probe (vocab strings whose BPE is
//                            themselves); on a miss the whole warp runs the
//                            exact multi-merge in registers (warp_engine.cuh)
//        longer              "deferred": a marker entry + a record
//   4. writes the tile's ids in order to its scratch SLOT (L2-resident) with
//      coalesced 16-B stores, its entry count, and the tile-local offsets of
//      the documents that start in it.
// Deferred segments (longer than SHORT_MAX: never in prose, which tops out at
// 14 bytes; digit/letter/newline runs) are then encoded by whole CTAs with the
// exact engine (engine.cuh) into the arena, and a second barrier follows.
// Phase B (place): CTA c owns a contiguous range of the round's tiles: it
// scans their counts, finds the range's output offset by a CTA-granular
// decoupled look-back (G units per round), copies the slots to the output
// (expanding deferred markers), fixes the documents' CSR offsets and discards
// the scratch lines from L2 without write-back.
#pragma once
#include "common.cuh"
#include "engine.cuh"
#include "warp_engine.cuh"

#ifndef GPUBPE_SEQ_ENGINE
#define GPUBPE_SEQ_ENGINE 1  // memo misses: 1 = warp_seq_bpe, 0 = warp_pack_bpe (multi-merge)
#endif
constexpr int WT = 512;         // bytes per warp tile (16 per lane)
constexpr int HALO = 32;        // bytes staged past the tile: any short segment ends inside
constexpr int LD = WT + HALO;   // staged bytes
constexpr int NGRP = LD / 16;   // 16-position groups whose cut bits are computed
#ifndef GPUBPE_NW
#define GPUBPE_NW 32
#endif
constexpr int NW = GPUBPE_NW;   // warps per CTA
constexpr int NT = NW * 32;     // threads per CTA
constexpr int SHORT_MAX = 32;   // longest segment encoded inside the tile loop
constexpr int GIANT_MIN = 4097; // deferred segments this long are giants (else a warp encodes them)
#ifndef GPUBPE_MEDIUM_MAX
#define GPUBPE_MEDIUM_MAX 1024
#endif
// deferred segments longer than this go to the CTA (or grid) engine with the giants:
// a warp's pass walks the segment 32 positions at a time, each step a few dependent
// L2 round trips, so a 2 KB digit run on a warp outlasts the whole giant pass
constexpr int MEDIUM_MAX = GPUBPE_MEDIUM_MAX < GIANT_MIN - 1 ? GPUBPE_MEDIUM_MAX : GIANT_MIN - 1;
#ifndef GPUBPE_FEW_MEDIUM_MAX
#define GPUBPE_FEW_MEDIUM_MAX 128
#endif
constexpr int FEW_MEDIUM_MAX = GPUBPE_FEW_MEDIUM_MAX < MEDIUM_MAX ? GPUBPE_FEW_MEDIUM_MAX : MEDIUM_MAX;
constexpr int CTA_GIANT_MAX = 64 << 10;  // with several giants in a round, one CTA each up to this length
constexpr int SLOT = WT + SHORT_MAX;  // scratch entries per tile (ids of segments starting in it)
#ifndef GPUBPE_UNIT_MAX
#define GPUBPE_UNIT_MAX 512
#endif
constexpr int UNIT_MAX = GPUBPE_UNIT_MAX;   // tiles per CTA per round in phase B
constexpr unsigned int MARK = 0x80000000u;  // scratch entry: deferred record index follows
constexpr int ARRIVE_MAX = 32;      // pieces of an overlapped host call (arrival words)
constexpr int ARRIVE_STRIDE = 32;   // u32 words between arrival words (one 128-B line each)
constexpr int RNG_MAX = 192;                // grids up to this many CTAs complete one-round calls
                                            // through per-range words instead of a grid barrier

// tile word: bits 0-15 entries, bit 16 has deferred markers, bits 17.. extra ids
// of the deferred segments beyond their one marker entry
#define TW_ENTRIES(w) ((uint32_t)((w) & 0xFFFFull))
#define TW_HASDEF(w) (((w) >> 16) & 1ull)
#define TW_EXTRA(w) ((w) >> 17)

struct PassCounters {
    unsigned long long n_segments;
    unsigned long long memo_hits;
    unsigned long long short_merges;
    unsigned long long medium_segments;
    unsigned long long giant_segments;
    unsigned long long giant_bytes;
    unsigned long long engine_passes;
};

// Per-call device state, zeroed before the call (each call zeroes the next
// call's slot; two slots alternate).  Hot words get their own 128-B lines.
struct EncodeState {
    unsigned long long actr[2];      // phase-A tile counters by round parity
    unsigned long long pad0[14];
    unsigned long long bar;          // low 32 bits: grid barrier arrivals; high 32 bits: deferred
                                     // segments recorded (read with the barrier, no extra round trip)
    unsigned long long pad1[15];
    unsigned long long ndef[2];      // deferred segments recorded, by round parity (multi-round
                                     // calls: a round's count independent of the next round's)
    unsigned long long rec_ctr;      // deferred records taken by warps (medium pass)
    unsigned long long rec_ctr2;     // deferred records scanned by CTAs (giant pass)
    unsigned long long arena_used;   // u32 words requested from the arena
    unsigned long long overflow;     // arena or record list overflowed: host re-runs
    unsigned long long n_ids;
    unsigned long long exit_ctr;     // CTAs that left the kernel (the last one fills EncodeParams.mirror)
    unsigned long long pad2[1];
    PassCounters c;
    unsigned long long rng[RNG_MAX];  // one-round calls: per placement range, tiles done << 40 | entries
};

// The results a host call needs, written by the last CTA into mapped pinned memory.
struct StateMirror {
    unsigned long long n_ids;
    unsigned long long overflow;
    PassCounters c;
    unsigned long long done;  // the call's tag, written last
};

struct DefRec {
    unsigned long long start;  // first byte of the segment
    unsigned int count;        // ids it encodes to
    unsigned int res;          // arena word offset of its ids
    unsigned long long dst;    // giants: output position, copied grid-wide after placement
    unsigned long long doc;    // a document at or before the one holding `start` (search hint)
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
    uint32_t *scratch;     // [2][R][SLOT] tile slots by round parity
    unsigned long long *tiles;   // [2][R] tile words by round parity
    unsigned long long *status;  // [n_rounds * grid] unit look-back words
    DefRec *recs;                // [rec_cap]
    unsigned long long rec_cap;
    uint32_t *arena;             // deferred-segment engine scratch + results
    unsigned long long arena_words;
    unsigned long long n_tiles;
    unsigned long long round_tiles;  // R
    unsigned int epoch;          // look-back tag
    int strict;
    int aligned;                 // bytes pointer is 16-B aligned
    int tile_bytes;              // wt: 128, 256 or 512 (host picks by input size)
    unsigned long long *gscr;    // grid-engine scratch: [0..7] scalars, [8..8+2*grid) per-CTA
    uint32_t *glist;             // [rec_cap] giant record indices of the round (count in gscr[4])
    const uint32_t *pretok;      // GPT-2 regex token-start bits (pretok.cu), null in the default mode
    const unsigned int *arrive;  // overlapped host calls: per-piece arrival words (DMA'd after each
                                 // piece of the input), else null -- a tile waits for its pieces
    unsigned long long piece;    // bytes per piece
    unsigned int arrive_tag;     // value of an arrived piece's word in this call
    StateMirror *mirror;         // host calls: results for the host (mapped pinned), else null
    unsigned long long mirror_tag;  // value of mirror->done once the results are complete
    unsigned long long *dbg;     // debug timestamps (GPUBPE_DEBUG & 8), else null
    int dbg_phase_a_only;        // GPUBPE_DEBUG & 16: profile phase A alone (output invalid)
};

// engine scratch for n tokens: tok, tok2 (u32) + pr, pr2 (uint2) + sel (u8)
#define ENGINE_BYTES(n) ((size_t)(n) * 25 + 64)
