// warp_engine.cuh -- exact BPE of SEVERAL short segments at once by one warp.
//
// The memo misses of a tile (segments of <= SHORT_MAX bytes that are not a
// vocab string whose BPE is itself; ~1.3% of prose segments) are packed
// back to back into the 32 lanes, lane j holding token j.  Each pass is one
// round of table probes plus register/shuffle work:
//   * strict mode (table not well-formed, or forced; one segment per pack):
//     the single leftmost minimum-rank pair -- the reference's own order
//     (engines.py:269-335), one merge per pass;
//   * well-formed tables (every rule using token T ranks above the rule
//     producing T; GPT-2 is): in every segment, all occurrences of the
//     segment's minimum rank (even offset inside runs of equal pairs: the
//     reference's leftmost-first pairing), plus any pair whose bounded
//     blocking walks succeed (no lower-rank merge can
//     reach it before its turn; a truncated walk only defers a merge).
// Pairs never span two packed segments: the last token of a segment has no
// pair and walks stop at segment ends, exactly as at the ends of a sequence.
#pragma once
#include "common.cuh"

#ifdef GPUBPE_DEBUG_STAMPS
#define ENG_MARK(k)                                                         \
    do {                                                                    \
        long long c_;                                                       \
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(c_));                  \
        eng_acc[k] += c_ - eng_prev;                                        \
        eng_prev = c_;                                                      \
    } while (0)
#else
#define ENG_MARK(k) do { } while (0)
#endif

#ifndef WALK_STEPS
#define WALK_STEPS 8
#endif

// Segment boundaries in lane order: bit j of `heads` marks a segment's first
// lane.  Last lane of the segment holding lane j (n = lanes in use).
__device__ __forceinline__ uint32_t seg_last_lane(uint32_t heads, uint32_t j, uint32_t n) {
    const uint32_t after = j >= 31 ? 0u : (heads & (0xFFFFFFFEu << j));
    return after ? (uint32_t)(__ffs(after) - 2) : n - 1;
}

// list[0..k): start | len << 16 of the segments (staged bytes sb), sum len <=
// 32.  Writes each segment's ids to sid[SI(start..)], tags the first with the
// count << 24.  Returns the passes run.
static __device__ uint32_t warp_pack_bpe(const DevTables &T, const uint32_t *base, const uint32_t *sbw,
                                  uint32_t *sid, const uint32_t *list, uint32_t k,
                                  bool strict, long long *eng_acc = nullptr) {
    const uint32_t lane = threadIdx.x & 31;
#ifdef GPUBPE_DEBUG_STAMPS
    long long eng_prev;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(eng_prev));
#endif
    const uint32_t ent_l = lane < k ? list[lane] : 0u;
    const uint32_t len_l = ent_l >> 16;
    uint32_t off = len_l;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL_MASK, off, o);
        if (lane >= (uint32_t)o) off += y;
    }
    const uint32_t total = __shfl_sync(FULL_MASK, off, 31);
    off -= len_l;  // first lane of segment `lane`
    const uint32_t heads0 = __reduce_or_sync(FULL_MASK, lane < k ? (1u << off) : 0u);
    // lane j: its segment, token, flags
    bool valid = lane < total;
    const uint32_t le = (lane >= 31) ? 0xFFFFFFFFu : ((2u << lane) - 1);
    const uint32_t seg = (uint32_t)__popc(heads0 & le) - 1;
    const uint32_t f = 31 - __clz(heads0 & le);
    const uint32_t ent = __shfl_sync(FULL_MASK, ent_l, seg & 31);
    uint32_t tok = valid ? base[sb_byte(sbw, (ent & 0xFFFFu) + lane - f)] : 0u;
    bool first = valid && ((heads0 >> lane) & 1u);
    bool last = valid && seg_last_lane(heads0, lane, total) == lane;
    uint32_t n = total;

    // initial pair probes and blocking ranks, one round
    uint32_t rk = GPUBPE_INF, nw = 0, rl = GPUBPE_INF, rr = GPUBPE_INF;
    {
        const uint32_t t1 = __shfl_down_sync(FULL_MASK, tok, 1);
        if (valid && !last) {
            const PairHit h = probe_pair(T, tok, t1);
            rk = h.rank;
            nw = h.nw;
        }
        if (valid && !strict) {
            rl = __ldg(&T.rl[tok]);
            rr = __ldg(&T.rr[tok]);
        }
    }
    ENG_MARK(0);  // setup + initial probes
    uint32_t np = 0;
    for (;;) {
        const bool live = valid && !last && rk != GPUBPE_INF;
        if (!__any_sync(FULL_MASK, live)) break;
        ++np;
        bool sel;
        if (strict) {
            const uint32_t m = __reduce_min_sync(FULL_MASK, live ? rk : GPUBPE_INF);
            const unsigned b = __ballot_sync(FULL_MASK, live && rk == m);
            sel = lane == (uint32_t)(__ffs(b) - 1);
        } else {
            // minimum rank of each packed segment: one REDUX when the pack holds
            // a single segment, else a forward segmented scan (rank in the low
            // 31 bits, head flag in bit 31: one shuffle per step) read at the
            // segment's last lane
            uint32_t segmin;
            if (k == 1) {
                segmin = __reduce_min_sync(FULL_MASK, live ? rk : GPUBPE_INF);
            } else {
                uint32_t x = (live ? min(rk, 0x7FFFFFFFu) : 0x7FFFFFFFu) | ((first || !valid) ? 0x80000000u : 0u);
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(FULL_MASK, x, o);
                    if (lane >= (uint32_t)o && !(x >> 31)) x = min(x, y & 0x7FFFFFFFu) | (y & 0x80000000u);
                }
                const uint32_t heads = __ballot_sync(FULL_MASK, first);
                const uint32_t sm = __shfl_sync(FULL_MASK, x, valid ? seg_last_lane(heads, lane, n) : lane) & 0x7FFFFFFFu;
                segmin = sm == 0x7FFFFFFFu ? GPUBPE_INF : sm;
            }
            ENG_MARK(1);  // segment minima
            // runs of equal pairs (identical tokens, e.g. "aaaa") pair up
            // leftmost-first: even offset inside the run
            const uint32_t rprev = __shfl_up_sync(FULL_MASK, rk, 1);
            const bool same = live && !first && rprev == rk;
            uint32_t s = lane;
            if (__any_sync(FULL_MASK, same)) {
                uint32_t st = (live && !same) ? lane : 0u;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(FULL_MASK, st, o);
                    if (lane >= (uint32_t)o) st = max(st, y);
                }
                s = st;
            }
            bool ok = live && ((lane - s) & 1u) == 0;
            const bool need = ok && rk != segmin;
            ENG_MARK(2);  // segmin + runs
            if (WALK_STEPS > 0 && __any_sync(FULL_MASK, need)) {
                // both blocking walks, one step of each per iteration: left
                // from the run start s, right from lane + 1
                uint32_t ql = s, qr = lane + 1;
                bool ldone = !need, lres = true, rdone = !need, rres = true;
#pragma unroll 1
                for (int it = 0; it < WALK_STEPS; ++it) {
                    const bool qfirst = __shfl_sync(FULL_MASK, first, ql & 31);
                    const uint32_t rrq = __shfl_sync(FULL_MASK, rr, ql & 31);
                    const uint32_t rkm = __shfl_sync(FULL_MASK, rk, (ql - 1) & 31);
                    const bool qlast = __shfl_sync(FULL_MASK, last, qr & 31);
                    const uint32_t rlq = __shfl_sync(FULL_MASK, rl, qr & 31);
                    const uint32_t rkq = __shfl_sync(FULL_MASK, rk, qr & 31);
                    if (!ldone) {
                        if (qfirst || rrq > rk) ldone = true;
                        else if (rkm < rk) { ldone = true; lres = false; }
                        else --ql;
                    }
                    if (!rdone) {
                        if (qlast || rlq > rk) rdone = true;
                        else if (rkq < rk) { rdone = true; rres = false; }
                        else ++qr;
                    }
                    if (!__any_sync(FULL_MASK, !(ldone && rdone) && !(ldone && !lres) && !(rdone && !rres))) break;
                }
                if (need) ok = ldone && lres && rdone && rres;
            } else if (need) {
                ok = false;  // no walks: only the segment minima merge this pass
            }
            sel = ok;
            ENG_MARK(3);  // walks
        }
        // apply: token j+1 disappears when pair j is selected
        const bool selprev = __shfl_up_sync(FULL_MASK, sel, 1) && lane > 0 && !first;
        const bool keep = valid && !selprev;
        const uint32_t newtok = sel ? nw : tok;
        const bool lastnext = __shfl_down_sync(FULL_MASK, last, 1);  // every lane shuffles
        const bool newlast = sel ? lastnext : last;
        const unsigned km = __ballot_sync(FULL_MASK, keep);
        const uint32_t n2 = __popc(km);
        const uint32_t src = lane < n2 ? __fns(km, 0, (int)lane + 1) : 0u;
        // token (< 2^24) and its three flags move in one shuffle
        const uint32_t packed = newtok | (first ? 1u << 24 : 0u) | (newlast ? 1u << 25 : 0u) | (sel ? 1u << 26 : 0u);
        const uint32_t moved = __shfl_sync(FULL_MASK, packed, src);
        valid = lane < n2;
        tok = moved & 0xFFFFFFu;
        first = valid && ((moved >> 24) & 1u);
        last = valid && ((moved >> 25) & 1u);
        const bool m2 = valid && ((moved >> 26) & 1u);
        const uint32_t rk_src = __shfl_sync(FULL_MASK, rk, src);
        const uint32_t nw_src = __shfl_sync(FULL_MASK, nw, src);
        const uint32_t rl_src = __shfl_sync(FULL_MASK, rl, src);
        const uint32_t rr_src = __shfl_sync(FULL_MASK, rr, src);
        const bool mnext = __shfl_down_sync(FULL_MASK, m2, 1);
        const uint32_t tnext = __shfl_down_sync(FULL_MASK, tok, 1);
        n = n2;
        rl = rl_src;
        rr = rr_src;
        ENG_MARK(4);  // compaction
        if (m2 && !strict) {  // loads in flight together with the pair probe below
            rl = __ldg(&T.rl[tok]);
            rr = __ldg(&T.rr[tok]);
        }
        if (valid && !last) {
            if (m2 || mnext) {
                const PairHit h = probe_pair(T, tok, tnext);
                rk = h.rank;
                nw = h.nw;
            } else {
                rk = rk_src;
                nw = nw_src;
            }
        } else {
            rk = GPUBPE_INF;
        }
        (void)__any_sync(FULL_MASK, rk == 0);  // (stamps: wait for the probe)
        ENG_MARK(5);  // re-probe
    }
    // write back: segment order is preserved by the compaction
    const uint32_t heads = __ballot_sync(FULL_MASK, first);
    const uint32_t le2 = (lane >= 31) ? 0xFFFFFFFFu : ((2u << lane) - 1);
    const uint32_t sg = (uint32_t)__popc(heads & le2) - 1;
    const uint32_t f2 = 31 - __clz(heads & le2);
    const uint32_t e2 = __shfl_sync(FULL_MASK, ent_l, sg & 31);
    const uint32_t p = e2 & 0xFFFFu;
    if (valid) sid[SI(p + lane - f2)] = tok;
    __syncwarp();
    if (first) {
        const uint32_t cnt = seg_last_lane(heads, lane, n) - lane + 1;
        sid[SI(p)] |= cnt << 24;
    }
    __syncwarp();
    return np;
}

// ------------------------------------------------------------------ sequential
//
// warp_seq_bpe: the same packs (list[0..k): start | len << 16, sum len <= 32,
// lane j = token j) merged the reference's own way -- every step merges, in
// every packed segment, the leftmost pair of minimum rank (engines.py:269-335)
// -- so it is exact for ANY table, well-formed or not.  Nothing moves between
// lanes: a merged pair's right token just dies (alive mask L), a token's right
// neighbour is the next live lane, and only the winner and the live token
// before it re-probe (two probes in flight per step).  A step is a segmented
// min, two ballots and one probe round, against the multi-merge pass's walks,
// compaction shuffles and rl/rr loads; its latency (one dependent probe) is
// what the tail of a latency-bound call waits for.  Returns the steps run.
static __device__ uint32_t warp_seq_bpe(const DevTables &T, const uint32_t *base, const uint32_t *sbw,
                                        uint32_t *sid, const uint32_t *list, uint32_t k,
                                        long long *eng_acc = nullptr) {
    const uint32_t lane = threadIdx.x & 31;
#ifdef GPUBPE_DEBUG_STAMPS
    long long eng_prev;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(eng_prev));
#endif
    const uint32_t ent_l = lane < k ? list[lane] : 0u;
    const uint32_t len_l = ent_l >> 16;
    uint32_t off = len_l;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL_MASK, off, o);
        if (lane >= (uint32_t)o) off += y;
    }
    const uint32_t total = __shfl_sync(FULL_MASK, off, 31);
    off -= len_l;  // first lane of segment `lane`
    const uint32_t heads = __reduce_or_sync(FULL_MASK, lane < k ? (1u << off) : 0u);
    const bool valid = lane < total;
    const uint32_t le = (lane >= 31) ? 0xFFFFFFFFu : ((2u << lane) - 1);
    const uint32_t seg = (uint32_t)__popc(heads & le) - 1;
    const uint32_t f = 31 - __clz(heads & le);               // first lane of my segment
    const uint32_t ha = heads & ~le;
    const uint32_t send = ha ? (uint32_t)(__ffs(ha) - 1) : total;  // one past my segment's last lane
    const uint32_t ent = __shfl_sync(FULL_MASK, ent_l, seg & 31);
    const uint32_t p0 = ent & 0xFFFFu;
    uint32_t tok = valid ? base[sb_byte(sbw, p0 + lane - f)] : 0u;
    uint32_t L = __ballot_sync(FULL_MASK, valid);  // live tokens
    uint32_t rk = GPUBPE_INF, nw = 0;
    {
        const uint32_t t1 = __shfl_down_sync(FULL_MASK, tok, 1);
        if (valid && lane + 1 < send) {
            const PairHit h = probe_pair(T, tok, t1);
            rk = h.rank;
            nw = h.nw;
        }
    }
    const uint32_t fmask = ~((1u << f) - 1);  // lanes >= f
    const bool head = (heads >> lane) & 1u;
    uint32_t steps = 0;
#ifdef GPUBPE_DEBUG_STAMPS
    (void)__any_sync(FULL_MASK, rk == 0);  // (stamps: wait for the probes)
#endif
    ENG_MARK(0);
    for (;;) {
        const bool alive = (L >> lane) & 1u;
        const bool live = alive && rk != GPUBPE_INF;
        if (!__any_sync(FULL_MASK, live)) break;
        ++steps;
        uint32_t m;
        if (k == 1) {
            m = __reduce_min_sync(FULL_MASK, live ? rk : GPUBPE_INF);
        } else if (k <= 4) {  // one reduction per segment
            m = GPUBPE_INF;
            for (uint32_t q = 0; q < k; ++q) {
                const uint32_t v = __reduce_min_sync(FULL_MASK, (live && seg == q) ? rk : GPUBPE_INF);
                if (seg == q) m = v;
            }
        } else {  // forward segmented min (head flag in bit 31), read at the segment's last lane
            uint32_t x = (live ? min(rk, 0x7FFFFFFFu) : 0x7FFFFFFFu) | ((head || !valid) ? 0x80000000u : 0u);
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(FULL_MASK, x, o);
                if (lane >= (uint32_t)o && !(x >> 31)) x = min(x, y & 0x7FFFFFFFu) | (y & 0x80000000u);
            }
            const uint32_t sm = __shfl_sync(FULL_MASK, x, valid ? send - 1 : lane) & 0x7FFFFFFFu;
            m = sm == 0x7FFFFFFFu ? GPUBPE_INF : sm;
        }
        ENG_MARK(1);
        // the leftmost candidate of each segment merges with the next live token
        const unsigned cand = __ballot_sync(FULL_MASK, live && rk == m);
        const unsigned mine = cand & fmask;
        const bool win = live && rk == m && (uint32_t)(__ffs(mine) - 1) == lane;
        const unsigned W = __ballot_sync(FULL_MASK, win);
        // each winner's right neighbour dies: the next live lane above it, found
        // for every winner at once by a carry through the dead lanes of ~L
        L &= ~((~L + (W << 1)) & L);
        if (win) tok = nw;
        ENG_MARK(2);
        // new right neighbours: the winners' and the tokens just before the winners
        const unsigned after = L & ~le;
        const uint32_t rn = after ? (uint32_t)(__ffs(after) - 1) : 32u;
        const bool still = (L >> lane) & 1u;
        const bool before_win = rn < 32 && ((W >> rn) & 1u);
        const uint32_t rt = __shfl_sync(FULL_MASK, tok, rn & 31);
#ifdef GPUBPE_DEBUG_STAMPS
        (void)__any_sync(FULL_MASK, rt == 0);
#endif
        ENG_MARK(3);
        if (still && (win || before_win)) {
            if (rn < send) {
                const PairHit h = probe_pair(T, tok, rt);
                rk = h.rank;
                nw = h.nw;
            } else {
                rk = GPUBPE_INF;
            }
        }
        if (!still) rk = GPUBPE_INF;
#ifdef GPUBPE_DEBUG_STAMPS
        (void)__any_sync(FULL_MASK, rk == 0);
#endif
        ENG_MARK(4);
    }
    // write back: each segment's live tokens in order, the first tagged with the count
    if ((L >> lane) & 1u) sid[SI(p0 + __popc(L & fmask & ((1u << lane) - 1)))] = tok;
    __syncwarp();
    if (valid && head) {
        const uint32_t smask = (send >= 32 ? 0xFFFFFFFFu : ((1u << send) - 1)) & fmask;
        sid[SI(p0)] |= (uint32_t)__popc(L & smask) << 24;
    }
    __syncwarp();
    return steps;
}
