// engine.cuh -- CTA-cooperative exact multi-merge BPE engine (K3 / K4 core).
//
// Runs greedy lowest-rank / leftmost BPE (reference: engines.py:269-335) on one
// token sequence with the whole CTA, in passes.  Each pass
//   1. reduces the minimum pair rank r_min (and its leftmost position),
//   2. selects pairs to merge this pass,
//   3. applies them with a double-buffered stream compaction and re-probes
//      only the pairs next to a merge.
// Selection rule:
//   * strict mode (table not well-formed, or forced): the pairs of rank r_min
//     (even offset in their runs) in position order, up to and including the
//     first whose merge creates a pair of rank <= r_min -- exactly the
//     reference's order (each is the leftmost global minimum when its turn
//     comes); at worst one merge per pass;
//   * well-formed tables (every rule using token T ranks above every rule
//     producing T; GPT-2 is): all pairs p with even offset inside their run of
//     equal-rank pairs and either rank == r_min, or a bounded "blocking walk"
//     proves no lower-rank merge can reach p before its turn:
//       left walk  from the run start j: stop OK at j==0 or rr[tok[j]] > r;
//                  fail if rank(j-1) < r; else j -= 1
//       right walk from j = p+1: stop OK at the last token or rl[tok[j]] > r;
//                  fail if rank(j) < r; else j += 1
//     (rl/rr = min rank of any rule with the token as left/right operand).
//     Merges in a well-formed table happen in non-decreasing rank order, the
//     walks show tokens p, p+1 are untouched until time r, and run parity is
//     the reference's leftmost-first pairing inside a run; the global-min run
//     starts are always selected, so every pass makes progress.  A truncated
//     walk only defers a merge.  DESIGN.md "Exactness" has the argument; the
//     fuzz tests check it against the oracle on random well-formed and
//     non-well-formed tables.
// Storage is generic (shared or global memory) so the same code serves the
// in-tile medium path (per-CTA scratch) and giant segments (arena).
#pragma once
#include "common.cuh"

#include <type_traits>

#ifndef ENGINE_WALK
#define ENGINE_WALK 64
#endif
// walk bound of the CTA and warp engines: a pass there is cheaper than on the grid,
// and digit runs walk far (r02n: 32 steps against 64: 1,000 x 6 KB digit documents
// 3.40 -> 3.05 ms; 16 or 8 steps cost more passes than they save)
#ifndef GROUP_WALK
#define GROUP_WALK 32
#endif
#ifndef WARP_WALK
#define WARP_WALK 16  // the warp engine's (its lanes walk in lock step: the longest walk sets the pace)
#endif

// A pair slot to be re-probed ({GPUBPE_INF, REPROBE}; a probe miss is {GPUBPE_INF, 0}).
#define REPROBE 0xFFFFFFFFu

struct EngineMem {
    uint32_t *tok, *tok2;  // tokens, double buffered
    uint2 *pr, *pr2;       // pair i: {rank, new token}, double buffered
    uint8_t *sel;          // pair i merged this pass
};

struct EngineShared {
    unsigned long long red[32];
    uint32_t scan[32];
    unsigned long long kmin;
    uint32_t carry;
};

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long u = __shfl_xor_sync(0xffffffffu, v, o);
        v = u < v ? u : v;
    }
    return v;
}

// Block-wide min of a u64 (all threads get the result).
__device__ __forceinline__ unsigned long long block_min_u64(unsigned long long v, EngineShared &sh) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_min_u64(v);
    __syncthreads();
    if (lane == 0) sh.red[wid] = v;
    __syncthreads();
    if (wid == 0) {
        unsigned long long x = lane < nw ? sh.red[lane] : ~0ull;
        x = warp_min_u64(x);
        if (lane == 0) sh.kmin = x;
    }
    __syncthreads();
    return sh.kmin;
}

// Block exclusive prefix sum of v; *total gets the block sum.
__device__ __forceinline__ uint32_t block_excl_sum(uint32_t v, EngineShared &sh, uint32_t *total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    __syncthreads();
    if (lane == 31) sh.scan[wid] = x;
    __syncthreads();
    if (wid == 0) {
        uint32_t s = lane < nw ? sh.scan[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < nw) sh.scan[lane] = s;  // inclusive warp totals
    }
    __syncthreads();
    uint32_t before = wid ? sh.scan[wid - 1] : 0;
    *total = sh.scan[nw - 1];
    return before + x - v;
}

// Block inclusive max-scan of v (values >= 0).
__device__ __forceinline__ uint32_t block_incl_max(uint32_t v, EngineShared &sh, uint32_t *total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x = max(x, y);
    }
    __syncthreads();
    if (lane == 31) sh.scan[wid] = x;
    __syncthreads();
    if (wid == 0) {
        uint32_t s = lane < nw ? sh.scan[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s = max(s, y);
        }
        if (lane < nw) sh.scan[lane] = s;
    }
    __syncthreads();
    uint32_t before = wid ? sh.scan[wid - 1] : 0;
    *total = sh.scan[nw - 1];
    return max(before, x);
}

// The blocking walks read their tokens, pair ranks and rl/rr in batches of
// WALK_BATCH steps (all loads of a batch in flight together: two dependent
// round trips per batch instead of per step), then decide the steps in order.
#ifndef WALK_BATCH
#define WALK_BATCH 4
#endif
__device__ __forceinline__ bool walk_left(const DevTables &T, const uint32_t *tok, const uint2 *pr,
                                          uint32_t j, uint32_t r, int max_steps = ENGINE_WALK) {
    for (int step = 0; step < max_steps; step += WALK_BATCH) {
        uint32_t t[WALK_BATCH], pk[WALK_BATCH], bl[WALK_BATCH];
#pragma unroll
        for (int k = 0; k < WALK_BATCH; ++k) {
            const bool in = (uint32_t)k < j;  // position j - k >= 1
            t[k] = (uint32_t)k <= j ? tok[j - k] : 0u;
            pk[k] = in ? pr[j - k - 1].x : GPUBPE_INF;
        }
#pragma unroll
        for (int k = 0; k < WALK_BATCH; ++k) bl[k] = (uint32_t)k <= j ? __ldg(&T.rr[t[k]]) : 0u;
#pragma unroll
        for (int k = 0; k < WALK_BATCH; ++k) {
            if (j == (uint32_t)k) return true;  // reached position 0
            if (bl[k] > r) return true;
            if (pk[k] < r) return false;
        }
        j -= WALK_BATCH;
    }
    return false;
}

__device__ __forceinline__ bool walk_right(const DevTables &T, const uint32_t *tok, const uint2 *pr,
                                           uint32_t j, uint32_t n, uint32_t r, int max_steps = ENGINE_WALK) {
    for (int step = 0; step < max_steps; step += WALK_BATCH) {
        uint32_t t[WALK_BATCH], pk[WALK_BATCH], bl[WALK_BATCH];
#pragma unroll
        for (int k = 0; k < WALK_BATCH; ++k) {
            const bool pair = j + k + 1 < n;  // token j + k has a right neighbour
            t[k] = pair ? tok[j + k] : 0u;
            pk[k] = pair ? pr[j + k].x : GPUBPE_INF;
        }
#pragma unroll
        for (int k = 0; k < WALK_BATCH; ++k) bl[k] = j + k + 1 < n ? __ldg(&T.rl[t[k]]) : 0u;
#pragma unroll
        for (int k = 0; k < WALK_BATCH; ++k) {
            if (j + k + 1 >= n) return true;
            if (bl[k] > r) return true;
            if (pk[k] < r) return false;
        }
        j += WALK_BATCH;
    }
    return false;
}

// Strict passes merge every r_min candidate up to the first "violation": a
// candidate (pair i of rank r_min, even offset in its run; M.sel marks them)
// whose merge creates a pair of rank <= r_min.  Its new token c is the same for
// all candidates (one rule); its left neighbour is c when pair i - 2 is a
// candidate (merged just before it), else token i - 1; its right neighbour is
// token i + 2 (nothing to its right has merged yet).  Up to that candidate each
// one is the leftmost global minimum when its turn comes.
#ifndef STRICT_MULTI
#define STRICT_MULTI 1
#endif
__device__ __forceinline__ bool strict_violates(const DevTables &T, const EngineMem &M, uint32_t i, uint32_t n,
                                                uint32_t rmin) {
    const uint32_t c = M.pr[i].y;
    bool v = false;
    if (i > 0) v = probe_pair(T, i >= 2 && M.sel[i - 2] ? c : M.tok[i - 1], c).rank <= rmin;
    if (!v && i + 2 < n) v = probe_pair(T, c, M.tok[i + 2]).rank <= rmin;
    return v;
}

// Cooperating groups the engine runs on: the whole CTA (giant segments) or
// one warp (medium segments, 32 encoded per CTA at a time).
struct BlockGroup {
    EngineShared &sh;
    __device__ uint32_t rank() const { return threadIdx.x; }
    __device__ uint32_t size() const { return blockDim.x; }
    __device__ void sync() const { __syncthreads(); }
    __device__ unsigned long long min_u64(unsigned long long v) const { return block_min_u64(v, sh); }
    __device__ uint32_t excl_sum(uint32_t v, uint32_t *total) const { return block_excl_sum(v, sh, total); }
    __device__ uint32_t incl_max(uint32_t v, uint32_t *total) const { return block_incl_max(v, sh, total); }
};

struct WarpGroup {
    __device__ uint32_t rank() const { return threadIdx.x & 31; }
    __device__ uint32_t size() const { return 32; }
    __device__ void sync() const { __syncwarp(); }
    __device__ unsigned long long min_u64(unsigned long long v) const { return warp_min_u64(v); }
    __device__ uint32_t excl_sum(uint32_t v, uint32_t *total) const {
        const uint32_t lane = threadIdx.x & 31;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        *total = __shfl_sync(0xffffffffu, x, 31);
        return x - v;
    }
    __device__ uint32_t incl_max(uint32_t v, uint32_t *total) const {
        const uint32_t lane = threadIdx.x & 31;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (uint32_t)o) x = max(x, y);
        }
        *total = __shfl_sync(0xffffffffu, x, 31);
        return x;
    }
};

// Token-level extras (tokens.cu only; EXT = false compiles them out):
//   trace  nullable; merge k of the run (in pass order, by position inside a
//          pass) stores (pass << 34) | (at the sequence start << 33) | (its right
//          token last << 32) | rank at trace[k] -- the reference's
//          merge-rank trace (engines.py:270,317-319) is this list in order when
//          passes merge one pair (strict mode), and sorted by rank otherwise
//          (a well-formed table merges in non-decreasing rank order);
//   fault  the reference's inject_compaction_fault (engines.py:252-266,
//          378-388): the first pass that can be corrupted merges the single
//          global-min pair ONE SLOT OFF (p+1, else p-1) with p's new token.
struct EngineExt {
    unsigned long long *trace;
    bool fault;
};

// Runs the engine on M.tok[0..n).  Returns the output length; *out points at
// the buffer holding the result.  Every thread of the group must call.
template <class G, bool EXT = false>
static __device__ uint32_t engine_run_g(const DevTables &T, EngineMem M, uint32_t n, bool strict, const G &g,
                                        uint32_t *passes_out, const uint32_t **out,
                                        EngineExt ext = EngineExt{nullptr, false}) {
    // kSplit (the CTA): the dependent chains of a pass -- blocking walks and the
    // re-probes after a merge -- run in loops of their own with no barrier inside,
    // so every thread's chains overlap the others' instead of each chunk of the
    // sequence waiting for its slowest walk or probe; the pass minimum is taken
    // while re-probing.  The warp keeps the fused loops (its lanes are in lock
    // step either way).
    constexpr bool kSplit = !std::is_same<G, WarpGroup>::value;
    constexpr int kWalk = std::is_same<G, WarpGroup>::value ? WARP_WALK : GROUP_WALK;
    const uint32_t nt = g.size(), me = g.rank();
    uint32_t passes = 0;
    const uint32_t n0 = n;
    bool fault = EXT && ext.fault;
    unsigned long long mine = ~0ull;  // (kSplit) this thread's min (rank, position) of the pass
    for (uint32_t b = 0; b < n; b += nt) {
        uint32_t i = b + me;
        if (i + 1 < n) {
            PairHit h = probe_pair(T, M.tok[i], M.tok[i + 1]);
            M.pr[i] = make_uint2(h.rank, h.nw);
            if (kSplit && h.rank != GPUBPE_INF) mine = min(mine, ((unsigned long long)h.rank << 32) | i);
        }
    }
    g.sync();
    while (n >= 2) {
        // 1. min (rank, position)
        if (!kSplit) {
            mine = ~0ull;
            for (uint32_t b = 0; b < n - 1; b += nt) {
                uint32_t i = b + me;
                if (i < n - 1) {
                    uint32_t r = M.pr[i].x;
                    if (r != GPUBPE_INF) {
                        unsigned long long k = ((unsigned long long)r << 32) | i;
                        mine = k < mine ? k : mine;
                    }
                }
            }
        }
        unsigned long long kmin = g.min_u64(mine);
        if (kmin == ~0ull) break;
        const uint32_t rmin = (uint32_t)(kmin >> 32);
        const uint32_t pmin = (uint32_t)kmin;
        // 2. selection
        bool corrupt = false;
        if (EXT && fault) {  // uniform across the group
            corrupt = pmin + 1 < n - 1 || pmin > 0;
            fault = !corrupt;
        }
        if (corrupt || (strict && !STRICT_MULTI)) {
            for (uint32_t b = 0; b < n; b += nt) {
                uint32_t i = b + me;
                if (i < n) M.sel[i] = (i == pmin);
            }
        } else if (strict) {
            // candidates: pairs of rank r_min at even offset inside their run, merged
            // in position order up to and including the first whose merge creates a
            // pair of rank <= r_min (the reference merges that pair next)
            uint32_t carry = 0;
            unsigned long long first = ~0ull;
            for (uint32_t b = 0; b < n; b += nt) {
                uint32_t i = b + me;
                bool pair = i + 1 < n;
                uint32_t r = pair ? M.pr[i].x : GPUBPE_INF;
                bool start = pair && (i == 0 || M.pr[i - 1].x != r);
                uint32_t chunk_max;
                uint32_t s = g.incl_max(start ? i : 0u, &chunk_max);
                s = max(s, carry);
                carry = max(carry, chunk_max);
                if (i < n) M.sel[i] = pair && r == rmin && ((i - s) & 1u) == 0;
            }
            g.sync();
            for (uint32_t b = 0; b < n; b += nt) {
                uint32_t i = b + me;
                if (i < n && M.sel[i] && strict_violates(T, M, i, n, rmin)) first = min(first, (unsigned long long)i);
            }
            const unsigned long long v = g.min_u64(first);
            if (v != ~0ull)
                for (uint32_t b = 0; b < n; b += nt) {
                    uint32_t i = b + me;
                    if (i < n && i > v) M.sel[i] = 0;
                }
        } else {
            uint32_t carry = 0;
            for (uint32_t b = 0; b < n; b += nt) {
                uint32_t i = b + me;
                bool pair = i + 1 < n;
                uint32_t r = pair ? M.pr[i].x : GPUBPE_INF;
                bool start = pair && (i == 0 || M.pr[i - 1].x != r);
                uint32_t chunk_max;
                uint32_t s = g.incl_max(start ? i : 0u, &chunk_max);
                s = max(s, carry);
                carry = max(carry, chunk_max);
                bool ok = pair && r != GPUBPE_INF && ((i - s) & 1u) == 0;
                if (kSplit) {
                    // walks deferred: run start kept in tok2 (free until the compaction)
                    if (i < n) M.tok2[i] = ok && r != rmin ? s : GPUBPE_INF;
                } else if (ok && r != rmin) {
                    ok = walk_left(T, M.tok, M.pr, s, r, kWalk) && walk_right(T, M.tok, M.pr, i + 1, n, r, kWalk);
                }
                if (i < n) M.sel[i] = ok;
            }
            if (kSplit)  // the same positions per thread as above: no barrier needed
                for (uint32_t i = me; i + 1 < n; i += nt) {
                    const uint32_t s = M.tok2[i];
                    if (s != GPUBPE_INF) {
                        const uint32_t r = M.pr[i].x;
                        M.sel[i] = walk_left(T, M.tok, M.pr, s, r, kWalk) &&
                                   walk_right(T, M.tok, M.pr, i + 1, n, r, kWalk);
                    }
                }
        }
        g.sync();
        if (EXT && corrupt) {
            if (me == 0) {
                const uint32_t q = pmin + 1 < n - 1 ? pmin + 1 : pmin - 1;
                M.sel[pmin] = 0;
                M.sel[q] = 1;
                M.pr[q] = make_uint2(rmin, M.pr[pmin].y);
            }
            g.sync();
        }
        // 3. apply + compact
        uint32_t carry = 0;
        for (uint32_t b = 0; b < n; b += nt) {
            uint32_t j = b + me;
            bool keep = j < n && !(j > 0 && M.sel[j - 1]);
            uint32_t total;
            uint32_t pos = carry + g.excl_sum(keep ? 1u : 0u, &total);
            carry += total;
            if (keep) {
                bool sj = M.sel[j];
                uint2 pj = (j + 1 < n) ? M.pr[j] : make_uint2(GPUBPE_INF, 0);
                // merges before j in this pass = tokens removed before j = j - pos
                if (EXT && sj && ext.trace)
                    ext.trace[(n0 - n) + (j - pos)] = ((unsigned long long)passes << 34) |
                                                      ((unsigned long long)(j == 0) << 33) |
                                                      ((unsigned long long)(j + 2 == n) << 32) | pj.x;
                uint32_t t = sj ? pj.y : M.tok[j];
                M.tok2[pos] = t;
                uint32_t jn = sj ? j + 2 : j + 1;
                if (jn < n) {
                    bool sn = M.sel[jn];
                    uint32_t tn = sn ? M.pr[jn].y : M.tok[jn];
                    if (sj || sn) {
                        if (kSplit) {
                            M.pr2[pos] = make_uint2(GPUBPE_INF, REPROBE);  // probed below
                        } else {
                            PairHit h = probe_pair(T, t, tn);
                            M.pr2[pos] = make_uint2(h.rank, h.nw);
                        }
                    } else {
                        M.pr2[pos] = pj;
                    }
                }
            }
        }
        g.sync();
        if (kSplit) {  // re-probe the pairs next to a merge; the next pass's minimum
            mine = ~0ull;
            for (uint32_t p = me; p + 1 < carry; p += nt) {
                uint2 v = M.pr2[p];
                if (v.x == GPUBPE_INF && v.y == REPROBE) {
                    const PairHit h = probe_pair(T, M.tok2[p], M.tok2[p + 1]);
                    v = make_uint2(h.rank, h.nw);
                    M.pr2[p] = v;
                }
                if (v.x != GPUBPE_INF) mine = min(mine, ((unsigned long long)v.x << 32) | p);
            }
            g.sync();
        }
        n = carry;
        uint32_t *tt = M.tok; M.tok = M.tok2; M.tok2 = tt;
        uint2 *pp = M.pr; M.pr = M.pr2; M.pr2 = pp;
        ++passes;
    }
    *passes_out = passes;
    *out = M.tok;
    return n;
}

// The CTA-wide engine (all threads of the CTA must call).
static __device__ uint32_t engine_run(const DevTables &T, EngineMem M, uint32_t n, bool strict,
                                      EngineShared &sh, uint32_t *passes_out, const uint32_t **out) {
    return engine_run_g(T, M, n, strict, BlockGroup{sh}, passes_out, out);
}
