// warp_engine.cuh -- exact BPE of one short segment (<= 32 tokens) by one warp.
//
// Lane j holds token j; pair j = (tok_j, tok_{j+1}) is probed by lane j.  Each
// pass applies the same selection rule as the CTA engine (engine.cuh: strict
// single global-min merge, or for well-formed tables every pair that is the
// global min or passes both blocking walks, with run parity), entirely in
// registers: run starts by a shuffle max-scan, walks by indexed shuffles,
// compaction by ballot + __fns + shuffle.  One round of table probes per pass
// (all lanes in parallel) instead of one dependent probe chain per merge.
#pragma once
#include "common.cuh"

#define FULL_MASK 0xffffffffu

__device__ __forceinline__ unsigned long long wmin64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long u = __shfl_xor_sync(FULL_MASK, v, o);
        v = u < v ? u : v;
    }
    return v;
}

// tok: this lane's token (lanes >= n ignored).  Writes the result to
// out[0..ret) (lane j writes out[j]); returns the output length.  All 32
// lanes must call.  *passes receives the number of passes.
__device__ __forceinline__ uint32_t warp_bpe(const DevTables &T, uint32_t tok, uint32_t n, bool strict,
                                             uint32_t *out, uint32_t *passes) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t rk = GPUBPE_INF, nw = 0;
    {
        uint32_t t1 = __shfl_down_sync(FULL_MASK, tok, 1);
        if (lane + 1 < n) {
            PairHit h = probe_pair(T, tok, t1);
            rk = h.rank;
            nw = h.nw;
        }
    }
    uint32_t np = 0;
    for (;;) {
        unsigned long long key = rk != GPUBPE_INF ? (((unsigned long long)rk << 32) | lane) : ~0ull;
        key = wmin64(key);
        if (key == ~0ull) break;
        ++np;
        const uint32_t rmin = (uint32_t)(key >> 32);
        bool sel;
        if (strict) {
            sel = lane == (uint32_t)key;
        } else {
            const bool pair = lane + 1 < n;
            const uint32_t rprev = __shfl_up_sync(FULL_MASK, rk, 1);
            const bool start = pair && (lane == 0 || rprev != rk);
            uint32_t s = start ? lane : 0u;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t v = __shfl_up_sync(FULL_MASK, s, o);
                if (lane >= (uint32_t)o) s = max(s, v);
            }
            bool ok = pair && rk != GPUBPE_INF && ((lane - s) & 1u) == 0;
            const bool need = ok && rk != rmin;
            if (__any_sync(FULL_MASK, need)) {
                const uint32_t rrv = lane < n ? __ldg(&T.rr[tok]) : GPUBPE_INF;
                const uint32_t rlv = lane < n ? __ldg(&T.rl[tok]) : GPUBPE_INF;
                // left walk from the run start s
                uint32_t j = s;
                bool done = !need, res = true;
                for (int it = 0; it < 32; ++it) {
                    uint32_t rrj = __shfl_sync(FULL_MASK, rrv, j & 31);
                    uint32_t rkm = __shfl_sync(FULL_MASK, rk, (j - 1) & 31);
                    if (!done) {
                        if (j == 0 || rrj > rk) done = true;
                        else if (rkm < rk) { done = true; res = false; }
                        else --j;
                    }
                    if (!__any_sync(FULL_MASK, !done)) break;
                }
                bool lres = res;
                // right walk from lane + 1
                j = lane + 1;
                done = !need;
                res = true;
                for (int it = 0; it < 32; ++it) {
                    uint32_t rlj = __shfl_sync(FULL_MASK, rlv, j & 31);
                    uint32_t rkj = __shfl_sync(FULL_MASK, rk, j & 31);
                    if (!done) {
                        if (j + 1 >= n || rlj > rk) done = true;
                        else if (rkj < rk) { done = true; res = false; }
                        else ++j;
                    }
                    if (!__any_sync(FULL_MASK, !done)) break;
                }
                if (need) ok = lres && res;
            }
            sel = ok;
        }
        // apply: token j+1 disappears when pair j is selected
        const bool selprev = __shfl_up_sync(FULL_MASK, sel, 1) && lane > 0;
        const bool keep = lane < n && !selprev;
        const uint32_t newtok = sel ? nw : tok;
        const unsigned km = __ballot_sync(FULL_MASK, keep);
        const uint32_t n2 = __popc(km);
        const uint32_t src = lane < n2 ? __fns(km, 0, (int)lane + 1) : 0u;
        const uint32_t t2 = __shfl_sync(FULL_MASK, newtok, src);
        const bool m2 = __shfl_sync(FULL_MASK, sel, src) && lane < n2;
        const uint32_t rk_src = __shfl_sync(FULL_MASK, rk, src);
        const uint32_t nw_src = __shfl_sync(FULL_MASK, nw, src);
        const bool mnext = __shfl_down_sync(FULL_MASK, m2, 1);
        tok = t2;
        n = n2;
        const uint32_t tnext = __shfl_down_sync(FULL_MASK, tok, 1);
        if (lane + 1 < n) {
            if (m2 || mnext) {
                PairHit h = probe_pair(T, tok, tnext);
                rk = h.rank;
                nw = h.nw;
            } else {
                rk = rk_src;
                nw = nw_src;
            }
        } else {
            rk = GPUBPE_INF;
        }
    }
    if (lane < n) out[lane] = tok;
    *passes = np;
    return n;
}
