// common.cuh -- device tables, hashes and probes shared by all encode kernels.
//
// Layout in HBM (built once per context by ctx.cu, L2-resident afterwards):
//   pair table   uint4 slots {left, right, rank, new}, power-of-two capacity at
//                <= 50% load, two-choice cuckoo: the two halves of fmix64 of
//                (left<<32)|right (the reference's hash, merge_table.py:49-57)
//                pick the two slots a rule may sit in (pair_slots).
//   rl / rr      per internal id: min rank of any rule with the id as LEFT /
//                RIGHT operand (INF if none) -- the blocking test of the exact
//                multi-merge pass.
//   jbits        65536-bit junction bitmap: bit (x<<8|y) set iff some reachable
//                rule joins a token ending in byte x to one starting with byte
//                y.  A byte pair outside J can never be merged across, so it
//                is an exact segment boundary.
//   base         byte -> internal id (byte_codec.py:97-111)
//   memo         uint4 slots {bytes0-3, bytes4-7, id, len | blob_off<<8} keyed
//                by the byte string of a vocab token whose BPE is itself;
//                blob holds bytes 8.. of tokens longer than 8 bytes as
//                zero-padded 8-byte chunks (blob_off counts chunks).
//   ext_id       internal -> external id (NULL when ids are used as-is).
#pragma once
#include <cstdint>

#define GPUBPE_INF 0xFFFFFFFFu
#define FULL_MASK 0xffffffffu

struct DevTables {
    const uint4 *pairs;
    uint32_t pair_mask;
    const uint32_t *rl;
    const uint32_t *rr;
    const uint32_t *jbits;
    const uint32_t *base;
    const uint4 *memo;
    uint32_t memo_mask;  // 0 with memo == nullptr disables the memo
    const unsigned long long *blob;
    const uint32_t *ext_id;
    int well_formed;  // exact multi-merge allowed (else one global-min merge per pass)
};

__host__ __device__ __forceinline__ uint64_t fmix64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xFF51AFD7ED558CCDull;
    x ^= x >> 33;
    x *= 0xC4CEB9FE1A85EC53ull;
    x ^= x >> 33;
    return x;
}

// Two-choice cuckoo slots of a pair: the low and high halves of one fmix64 of
// (left << 32) | right (the reference's key and hash, merge_table.py:49-57).
// Every rule sits in one of its two slots, so a probe is two independent
// 16-byte loads -- one round trip for hits and misses alike, no chains.
struct PairSlots {
    uint32_t a, b;
};
__host__ __device__ __forceinline__ PairSlots pair_slots(uint32_t l, uint32_t r, uint32_t mask) {
    const uint64_t h = fmix64(((uint64_t)l << 32) | r);
    return PairSlots{(uint32_t)h & mask, (uint32_t)(h >> 32) & mask};
}

// Memo hash over a byte string given as 8-byte little-endian chunks:
// multiplicative (one 64-bit multiply per chunk, most strings are one chunk);
// the slot is taken from the top bits (memo_slot_of), which every input bit
// reaches.
__host__ __device__ __forceinline__ uint64_t memo_hash_step(uint64_t h, uint64_t chunk) {
    return (h ^ chunk) * 0x9E3779B97F4A7C15ull;
}
__host__ __device__ __forceinline__ uint64_t memo_hash_init(uint32_t len) {
    return (uint64_t)(len + 1) * 0xC2B2AE3D27D4EB4Full;
}
__host__ __device__ __forceinline__ uint32_t memo_slot_of(uint64_t h, uint32_t mask) {
    return (uint32_t)(h >> 40) & mask;
}

#ifdef __CUDACC__

// Skewed shared-memory layouts of a warp tile.  Lane L owns bytes [16L,
// 16L+16), so plain layouts put every lane's k-th slot in the same bank
// (16-way conflicts for u32 slots, 8-way for byte words).  One pad word per
// 16 slots / per 4 byte-words spreads the lanes over all 32 banks.
__host__ __device__ constexpr uint32_t SI(uint32_t p) { return p + (p >> 4); }  // slot of position p
__host__ __device__ constexpr uint32_t SW(uint32_t w) { return w + (w >> 2); }  // word of byte-word w
__device__ __forceinline__ uint32_t sb_byte(const uint32_t *sbw, uint32_t p) {
    return (sbw[SW(p >> 2)] >> (8 * (p & 3))) & 0xFFu;
}

struct PairHit {
    uint32_t rank;  // GPUBPE_INF on miss
    uint32_t nw;
};

__device__ __forceinline__ PairHit probe_pair(const DevTables &T, uint32_t l, uint32_t r) {
    const PairSlots ps = pair_slots(l, r, T.pair_mask);
    const uint4 a = __ldg(&T.pairs[ps.a]);
    const uint4 b = __ldg(&T.pairs[ps.b]);
    if (a.x == l && a.y == r) return PairHit{a.z, a.w};
    if (b.x == l && b.y == r) return PairHit{b.z, b.w};
    return PairHit{GPUBPE_INF, 0};
}

__device__ __forceinline__ bool is_junction(const uint32_t *jb, uint32_t x, uint32_t y) {
    uint32_t k = (x << 8) | y;
    return (__ldg(&jb[k >> 5]) >> (k & 31)) & 1u;
}

__device__ __forceinline__ uint32_t out_id(const DevTables &T, uint32_t v) {
    return T.ext_id ? __ldg(&T.ext_id[v]) : v;
}

#endif
