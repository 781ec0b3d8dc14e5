// kernels.cu -- the fused encode kernel (see kernels.cuh for the pipeline).
//
// Semantics restated from the reference (paths under /root/reference/pkg):
//   per-byte base ids             src/lanebpe/chunker.py:95-98
//   fixed-offset chunk cuts when   src/lanebpe/chunker.py:42-53, 139-144
//   len > max_seq_len
//   greedy min-rank / leftmost     src/lanebpe/engines.py:269-335
//   ordered reassembly             src/lanebpe/chunker.py:166-179
// Segment boundaries (junction bitmap, document starts, chunk cuts) are exact
// cut points: no merge of the reference can ever span them, so segments are
// encoded independently and concatenated in order.
#include <cuda_runtime.h>

#include <cuda/atomic>

#include "kernels.cuh"

// ------------------------------------------------------------------ smem

struct __align__(16) WarpSmem {
    union {
        struct {
            uint32_t sbw[SW((LD + 16) / 4) + 1];  // staged bytes, skewed words (+ slack for 8-B reads)
            uint32_t miss[WT / 2 + 2];      // memo misses: start | len << 16
        } a;
        uint32_t outbuf[SLOT];              // scratch entries in output order
    } u;
    uint32_t sid[SI(SLOT) + 2];  // at SI(p): ids of the segment starting at p; first tagged count << 24
                          // (0xFF: deferred, record index in the next slot)
    uint16_t seg[WT];           // starts of the segments beginning in the tile, in order
    uint32_t cm[NGRP / 2 + 1];  // cut bits, position k = cut before byte a + k
    uint32_t n_miss, n_def;
    unsigned long long dl_arena;  // deferred pass: this warp's arena offset broadcast
};

struct CtaSmem {
    uint32_t jb[2048];  // junction bitmap
    uint32_t base[256];
    EngineShared es;
    unsigned long long bcast[4];
    unsigned long long seen[2];     // ndef[] by parity as of this CTA's last read (thread 0)
    uint32_t arrived, poll_lock;    // overlapped host calls: pieces seen arrived; poller lock
    unsigned long long red[NW][4];  // per-warp partial sums (no 64-bit shared atomics: CAS loops)
    PassCounters pc;
    unsigned long long tb[UNIT_MAX];  // phase B: tile output offsets inside the unit
    unsigned long long tw[UNIT_MAX];  // phase B: tile words
    WarpSmem w[NW];
};

struct WarpCtx {
    long long dcur;  // document cursor: tiles of one warp are increasing
    unsigned long long n_segments, memo_hits, short_merges, engine_passes;  // per lane
};

// ------------------------------------------------------------------ helpers

// Relaxed gpu-scope accesses as plain PTX (libcu++'s atomic_ref adds a
// "local memory?" test and a local-memory fallback path to every access).
__device__ __forceinline__ void st_relaxed(unsigned long long *w, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(w), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed(unsigned long long *w) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(w) : "memory");
    return v;
}
// Relaxed polling: an acquire load would invalidate the SM's L1 (CCTL.IVALL)
// on every iteration and stall the other warps' L1/shared-memory traffic.
__device__ __forceinline__ unsigned int ld_relaxed_u32(unsigned int *w) {
    unsigned int v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(w) : "memory");
    return v;
}

__device__ __forceinline__ void red_release_add(unsigned long long *w, unsigned long long v) {
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(w), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Debug cycle stamp k of tile t after value v is available (GPUBPE_DEBUG & 8).
#ifdef GPUBPE_DEBUG_STAMPS
#define TSTAMP(k, v)                                                                     \
    do {                                                                                 \
        if (P.dbg && t < 2048) {                                                         \
            uint32_t d_;                                                                 \
            asm volatile("mov.b32 %0, %1;" : "=r"(d_) : "r"((uint32_t)(v)));            \
            __syncwarp();                                                                \
            long long c_;                                                                \
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(c_) : "r"(d_));               \
            if (lane == 0) P.dbg[16384 + 8 * t + (k)] = (unsigned long long)(c_ - dbg_c0); \
        }                                                                                \
    } while (0)
#else
#define TSTAMP(k, v) do { } while (0)
#endif

__device__ __forceinline__ uint4 ldg_stream(const uint4 *p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

// Smallest structural cut (doc end or chunk cut) strictly after p; doc d holds p.
__device__ __forceinline__ long long next_struct_cut(const EncodeParams &P, long long d, long long p) {
    long long s = __ldg(&P.doc_offs[d]), e = __ldg(&P.doc_offs[d + 1]);
    long long cut = e;
    if ((unsigned long long)(e - s) > P.max_seq_len) {
        long long cb = (long long)P.chunk_budget;
        long long c = s + ((p - s) / cb + 1) * cb;
        if (c < cut) cut = c;
    }
    return cut;
}

// Warp: last document d with offs[d] <= p (p < n_bytes), i.e. the non-empty
// document holding byte p.  32-ary search in [lo, n_docs), offs[lo] <= p.
__device__ long long warp_doc_from(const long long *offs, long long lo, unsigned long long n_docs,
                                   long long p) {
    const int lane = threadIdx.x & 31;
    long long hi = (long long)n_docs - 1;
    if (lo < hi && __ldg(&offs[lo + 1]) > p) return lo;  // still inside the last tile's document
    {   // the next 31 documents first: tiles of one warp move forward slowly
        const long long idx = lo + lane;
        const bool ok = idx <= hi && __ldg(&offs[idx]) <= p;
        const unsigned m = __ballot_sync(FULL_MASK, ok);
        if (m != FULL_MASK) return lo + 31 - __clz(m);
        lo += 31;
    }
    while (hi > lo) {
        const long long step = (hi - lo + 32) / 32;
        const long long idx = lo + (long long)lane * step;
        const bool ok = idx <= hi && __ldg(&offs[idx]) <= p;
        const unsigned m = __ballot_sync(FULL_MASK, ok);  // lane 0 is always true
        const int last = 31 - __clz(m);
        lo = lo + (long long)last * step;
        hi = min(hi, lo + step - 1);
    }
    return lo;
}

// GPT-2 regex mode: a pre-token starts at byte p.
__device__ __forceinline__ bool pretok_cut(const EncodeParams &P, long long p) {
    return P.pretok && ((__ldg(&P.pretok[p >> 5]) >> (p & 31)) & 1u);
}

// CTA: first p in [lo, hi) whose cut slot is a junction miss (or a pre-token
// start in GPT-2 regex mode), else hi.
__device__ long long cta_first_nonjunction(const EncodeParams &P, const uint32_t *jb, long long lo,
                                           long long hi, EngineShared &sh) {
    for (long long b = lo; b < hi; b += 16 * NT) {
        const long long p0 = b + 16 * (long long)threadIdx.x;
        unsigned long long k = ~0ull;
        if (p0 < hi) {
            uint32_t x = __ldg(&P.bytes[p0 - 1]);
            const long long pe = min(p0 + 16, hi);
            for (long long p = p0; p < pe; ++p) {
                const uint32_t y = __ldg(&P.bytes[p]);
                const uint32_t idx = (x << 8) | y;
                if (!((jb[idx >> 5] >> (idx & 31)) & 1u) || pretok_cut(P, p)) { k = (unsigned long long)p; break; }
                x = y;
            }
        }
        const unsigned long long m = block_min_u64(k, sh);
        if (m != ~0ull) return (long long)m;
    }
    return hi;
}

// Cut bits of the 8 positions of group g (position k: cut before byte 8g + k).
__device__ __forceinline__ uint32_t group8_cuts(const uint32_t *jb, const uint32_t *sbw, int g, uint32_t prevb) {
    uint32_t x = g ? sb_byte(sbw, 8 * g - 1) : prevb;
    const uint32_t w[2] = {sbw[SW(2 * g)], sbw[SW(2 * g + 1)]};
    uint32_t m = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t y = (w[k >> 2] >> (8 * (k & 3))) & 0xFFu;
        const uint32_t idx = (x << 8) | y;
        m |= ((jb[idx >> 5] >> (idx & 31)) & 1u) << k;
        x = y;
    }
    return ~m & 0xFFu;
}

// First cut in [q, lim], lim - q < 32; -1 if none.
__device__ __forceinline__ int next_cut(const uint32_t *cm, int q, int lim) {
    int w = q >> 5;
    uint32_t bits = cm[w] & (0xFFFFFFFFu << (q & 31));
    if (!bits) {
        ++w;
        if (w * 32 > lim) return -1;
        bits = cm[w];
        if (!bits) return -1;
    }
    const int c = w * 32 + __ffs(bits) - 1;
    return c <= lim ? c : -1;
}

// 8 bytes of the staged tile starting at byte p (little endian).
__device__ __forceinline__ unsigned long long sb_load8(const uint32_t *sbw, uint32_t p) {
    const uint32_t w = p >> 2;
    const uint32_t sh = (p & 3) * 8;
    const uint32_t w0 = sbw[SW(w)], w1 = sbw[SW(w + 1)], w2 = sbw[SW(w + 2)];
    const uint32_t lo = __funnelshift_r(w0, w1, sh);
    const uint32_t hi = __funnelshift_r(w1, w2, sh);
    return ((unsigned long long)hi << 32) | lo;
}

// The low n bytes of v (n >= 1; all of v from 8 on).
__device__ __forceinline__ unsigned long long low_bytes(unsigned long long v, uint32_t n) {
    return v & (~0ull >> (64 - 8 * min(n, 8u)));
}

// Memo lookup of staged bytes [p, p + len), 2 <= len <= SHORT_MAX: the id, or
// INF when the string is not a memoised vocab token (a vocab string whose BPE
// is itself).  Linear probing from the hash's slot to an empty one.
__device__ uint32_t memo_lookup(const DevTables &T, const uint32_t *sb, uint32_t p, uint32_t len) {
    const unsigned long long c0 = low_bytes(sb_load8(sb, p), len);
    unsigned long long h = memo_hash_step(memo_hash_init(len), c0);
    // bytes 8..15 are kept for the verification (strings of 9..16 bytes: no reload)
    const unsigned long long c1 = len > 8 ? low_bytes(sb_load8(sb, p + 8), len - 8) : 0ull;
    if (len > 8) h = memo_hash_step(h, c1);
    for (uint32_t c = 16; c < len; c += 8) h = memo_hash_step(h, low_bytes(sb_load8(sb, p + c), len - c));
    uint32_t slot = memo_slot_of(h, T.memo_mask);
    for (;;) {
        const uint4 e = __ldg(&T.memo[slot]);
        if (e.w == 0) return GPUBPE_INF;
        if ((e.w & 0xFFu) == len && e.x == (uint32_t)c0 && e.y == (uint32_t)(c0 >> 32)) {
            bool eq = true;
            if (len > 8) {
                const unsigned long long *tail = T.blob + (e.w >> 8);
                eq = __ldg(&tail[0]) == c1;
                for (uint32_t c = 16, k = 1; c < len; c += 8, ++k)
                    eq &= __ldg(&tail[k]) == low_bytes(sb_load8(sb, p + c), len - c);
            }
            if (eq) return e.z;
        }
        slot = (slot + 1) & T.memo_mask;
    }
}

// Warp decoupled look-back: publishes this tile's total, returns its base.
#define LB_AGG 1ull
#define LB_INC 2ull
#define LB_VALUE_MASK ((1ull << 42) - 1)

__device__ __forceinline__ unsigned long long warp_lookback(unsigned long long *status, unsigned long long t,
                                                            unsigned long long total, unsigned int epoch) {
    const int lane = threadIdx.x & 31;
    const unsigned long long tag = (unsigned long long)epoch << 44;
    if (t == 0) {
        if (lane == 0) st_relaxed(&status[0], tag | (LB_INC << 42) | total);
        return 0;
    }
    if (lane == 0) st_relaxed(&status[t], tag | (LB_AGG << 42) | total);
    unsigned long long excl = 0;
    long long pos = (long long)t - 1;
    for (;;) {
        const long long j = pos - lane;
        unsigned long long v, flag;
        if (j >= 0) {
            for (;;) {
                v = ld_relaxed(&status[j]);
                flag = ((v >> 44) == epoch) ? ((v >> 42) & 3ull) : 0ull;
                if (flag) break;
                __nanosleep(32);
            }
        } else {
            v = LB_INC << 42;
            flag = LB_INC;
        }
        const unsigned inc = __ballot_sync(FULL_MASK, flag == LB_INC);
        const int stop = inc ? __ffs(inc) - 1 : 31;
        unsigned long long val = lane <= stop ? (v & LB_VALUE_MASK) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(FULL_MASK, val, o);
        excl += val;
        if (inc) break;
        pos -= 32;
    }
    if (lane == 0) st_relaxed(&status[t], tag | (LB_INC << 42) | (excl + total));
    return excl;
}

// Cut bits of the 16 positions owned by lane L (explicit 16-bit load: the
// shift-and-mask form was once widened by the compiler into a misaligned
// 32-bit shared load at cm + 2L).
__device__ __forceinline__ uint32_t lane_cuts(const WarpSmem &S, int L) {
    return reinterpret_cast<const uint16_t *>(S.cm)[L];
}

// Count of the scratch entries of the segment whose sid tag is v.
__device__ __forceinline__ uint32_t seg_entries(uint32_t v) {
    const uint32_t cc = v >> 24;
    return cc == 0xFFu ? 1u : cc;
}

__device__ __forceinline__ void l2_discard(const void *p) {
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

// ------------------------------------------------------------------ phase A

// Encode tile t (bytes [t * wt, t * wt + wt)) into scratch slot `slot` (see
// kernels.cuh, phase A).  The segments starting in the tile are gathered
// into a position-ordered list and dealt round-robin to the lanes, so every
// lane handles ~1/32 of them (a warp's latency is its slowest lane's chain).
__device__ __noinline__ uint32_t encode_tile(const EncodeParams &P, CtaSmem &C, WarpSmem &S, unsigned long long t,
                                             unsigned long long slot, WarpCtx &X) {
    const int lane = threadIdx.x & 31;
    const DevTables &T = P.T;
    const int wt = P.tile_bytes;
    const int ld = wt + HALO;
    const long long N = (long long)P.n_bytes;
    const long long a = (long long)t * wt;
    const int nst = (int)min((long long)ld, N - a);
    const int nin = min(wt, nst);
    const bool last = a + wt >= N;
    uint32_t *sb = S.u.a.sbw;
    uint32_t c_seg = 0, c_memo = 0, c_miss = 0, c_pass = 0;

    // ---- 0. overlapped host call: wait until the pieces holding bytes
    //         [a - 1, a + nst) have arrived (their words are DMA'd after them;
    //         no SM reads a piece before its word, so no stale line can exist)
    //         One global poller per CTA at a time (a shared-memory lock); the
    //         other warps watch the CTA's arrived mask in shared memory.
    if (P.arrive) {
        if (lane == 0) {
            const bool one = P.piece >= P.n_bytes;  // (one piece: no division)
            const uint32_t k0 = one ? 0u : (uint32_t)((unsigned long long)(a > 0 ? a - 1 : 0) / P.piece);
            const uint32_t k1 = one ? 0u : (uint32_t)((unsigned long long)(a + nst - 1) / P.piece);
            const uint32_t need = (k1 >= 31 ? 0xFFFFFFFFu : ((2u << k1) - 1)) & ~((1u << k0) - 1);
            volatile uint32_t *arrived = &C.arrived;
            while ((*arrived & need) != need) {
                if (atomicCAS(&C.poll_lock, 0u, 1u) == 0u) {
                    uint32_t m = *arrived;
                    for (uint32_t k = k0; k <= k1; ++k)
                        if (!((m >> k) & 1u) &&
                            ld_relaxed_u32(const_cast<unsigned int *>(&P.arrive[ARRIVE_STRIDE * k])) == P.arrive_tag)
                            m |= 1u << k;
                    atomicOr(&C.arrived, m);
                    atomicExch(&C.poll_lock, 0u);
                    if ((m & need) == need) break;
                }
                __nanosleep(256);
            }
        }
        if (P.dbg && lane == 0) atomicMax(&P.dbg[36864 + 4 * blockIdx.x + 3], gtimer());
        __syncwarp();
        asm volatile("" ::: "memory");
    }
    // ---- 1. stage the tile and its halo (16-B loads, both rounds in flight)
    if (P.aligned && nst == ld) {
        const uint4 *src = reinterpret_cast<const uint4 *>(P.bytes + a);
        const int nv = ld / 16;
        uint4 v0 = make_uint4(0, 0, 0, 0), v1 = v0;
        if (lane < nv) v0 = ldg_stream(src + lane);
        if (lane + 32 < nv) v1 = ldg_stream(src + 32 + lane);
        if (lane < nv) {
            uint32_t *d = sb + SW(4 * lane);  // a lane's 4 words are contiguous after skewing
            d[0] = v0.x; d[1] = v0.y; d[2] = v0.z; d[3] = v0.w;
        }
        if (lane + 32 < nv) {
            uint32_t *d = sb + SW(4 * (32 + lane));
            d[0] = v1.x; d[1] = v1.y; d[2] = v1.z; d[3] = v1.w;
        }
    } else {
        uint8_t *b8 = reinterpret_cast<uint8_t *>(sb);
#pragma unroll 1
        for (int k = lane; k < ld; k += 32) b8[4 * SW(k >> 2) + (k & 3)] = k < nst ? __ldg(&P.bytes[a + k]) : 0;
    }
#ifdef GPUBPE_DEBUG_STAMPS
    long long dbg_c0 = 0;
    if (P.dbg) asm volatile("mov.u64 %0, %%clock64;" : "=l"(dbg_c0));
#endif
    const uint32_t prevb = a > 0 ? __ldg(&P.bytes[a - 1]) : 0u;
    if (lane == 0) {
        S.n_miss = 0;
        S.n_def = 0;
    }
    __syncwarp();
    TSTAMP(0, sb[SW(4 * lane)] + prevb);

    // ---- 2. cut bits: junction misses, start and end of input
    //         (8 positions per lane, so small tiles use 20 lanes, not 10; four
    //         lanes' bytes make one word; one zero word past the staged bytes)
    {
        const int ng = ld / 8;
#pragma unroll 1
        for (int i = 0; 32 * i < ng + 4; ++i) {
            const int g = lane + 32 * i;
            uint32_t mg = 0;
            if (g < ng) {
                mg = group8_cuts(C.jb, sb, g, prevb);
                const int p0 = 8 * g;
                if (p0 >= nst) mg = 0;
                else if (p0 + 8 > nst) mg &= (1u << (nst - p0)) - 1;
                if (a + nst == N && nst >= p0 && nst < p0 + 8) mg |= 1u << (nst - p0);
                if (g == 0 && a == 0) mg |= 1u;
            }
            uint32_t v = mg << (8 * (lane & 3));
            v |= __shfl_xor_sync(FULL_MASK, v, 1);
            v |= __shfl_xor_sync(FULL_MASK, v, 2);
            if (!(lane & 3) && (g >> 2) < NGRP / 2 + 1) S.cm[g >> 2] = v;
        }
    }
    __syncwarp();
    if (P.pretok) {  // GPT-2 regex mode: pre-token starts are cuts too
        const int nwords = (nst + 31) >> 5;
        if (lane < nwords) S.cm[lane] |= __ldg(&P.pretok[(a >> 5) + lane]);
        __syncwarp();
    }
    TSTAMP(1, S.cm[lane & 15]);

    // ---- 3. document starts and chunk cuts inside the staged bytes
    long long dc = 0;  // document holding byte a
    if (P.n_docs > 1) dc = X.dcur = warp_doc_from(P.doc_offs, X.dcur, P.n_docs, a);
    // inner: the staged bytes lie strictly inside document dc, with no chunk cut
    // among them -- no cut to add here and no document offset to record (step 8)
    bool inner = false;
    if (P.n_docs > 1 || (unsigned long long)N > P.max_seq_len) {
        const long long ds = __ldg(&P.doc_offs[dc]), de = __ldg(&P.doc_offs[dc + 1]);
        if (ds < a && de >= a + nst) {
            inner = true;
            if ((unsigned long long)(de - ds) > P.max_seq_len) {  // fixed-offset chunks: the next cut
                const unsigned long long cb = P.chunk_budget, num = (unsigned long long)(a - ds);
                unsigned long long r;
                if ((cb & (cb - 1)) == 0) r = num & (cb - 1);
                else if ((num >> 32) == 0 && (cb >> 32) == 0) r = (uint32_t)num % (uint32_t)cb;
                else r = num % cb;
                if (r == 0 || cb - r < (unsigned long long)nst) inner = false;
            }
        }
    }
    if (!inner && (P.n_docs > 1 || (unsigned long long)N > P.max_seq_len)) {
#pragma unroll 1
        for (long long d0 = dc;; d0 += 32) {
            const long long d = d0 + lane;
            bool in = false;
            if (d < (long long)P.n_docs) {
                const long long s = __ldg(&P.doc_offs[d]);
                if (s < a + nst) {
                    in = true;
                    if (s >= a) atomicOr(&S.cm[(s - a) >> 5], 1u << ((s - a) & 31));
                    const long long e = __ldg(&P.doc_offs[d + 1]);
                    if ((unsigned long long)(e - s) > P.max_seq_len) {
                        const long long cb = (long long)P.chunk_budget;
                        long long k = 1;
                        if (s < a) {  // first chunk cut at or after a (64-bit division only when needed)
                            const unsigned long long num = (unsigned long long)(a - s + cb - 1);
                            if ((cb & (cb - 1)) == 0) k = (long long)(num >> (63 - __clzll(cb)));
                            else if ((num >> 32) == 0 && ((unsigned long long)cb >> 32) == 0)
                                k = (long long)((uint32_t)num / (uint32_t)cb);
                            else k = (long long)(num / (unsigned long long)cb);
                        }
                        if (k < 1) k = 1;
#pragma unroll 1
                        for (long long c = s + k * cb; c < e && c < a + nst; c += cb)
                            atomicOr(&S.cm[(c - a) >> 5], 1u << ((c - a) & 31));
                    }
                }
            }
            if (__ballot_sync(FULL_MASK, in) != FULL_MASK) break;
        }
        __syncwarp();
    }

    // ---- 4. position-ordered list of the segments starting in the tile
    uint32_t nseg;
    {
        uint32_t mine = lane_cuts(S, lane);
        const int p0 = 16 * lane;
        if (p0 >= nin) mine = 0;
        else if (p0 + 16 > nin) mine &= (1u << (nin - p0)) - 1;
        const uint32_t c = __popc(mine);
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL_MASK, incl, o);
            if (lane >= o) incl += y;
        }
        nseg = __shfl_sync(FULL_MASK, incl, 31);
        uint32_t k = incl - c;
#pragma unroll 1
        for (uint32_t bits = mine; bits; bits &= bits - 1) S.seg[k++] = (uint16_t)(p0 + __ffs(bits) - 1);
    }
    __syncwarp();

    // ---- 5. classify and look up: length 1 -> base id, 2..SHORT_MAX -> memo
    //         (hash, probe and compare in one pass: the other warps of the SM
    //         cover the probe's latency), longer -> deferred
    const bool use_memo = T.memo_mask != 0;
#pragma unroll 1
    for (uint32_t i = lane; i < nseg; i += 32) {
        const int p = S.seg[i];
        // its end: the next segment's start (the list holds every cut in the tile),
        // past the tile the cut bits; -1 beyond SHORT_MAX
        int e;
        if (i + 1 < nseg) {
            e = S.seg[i + 1];
            if (e - p > SHORT_MAX) e = -1;
        } else {
            e = next_cut(S.cm, p + 1, p + SHORT_MAX);
        }
        ++c_seg;
        if (e < 0) {  // longer than SHORT_MAX: deferred to the CTA engine
            const unsigned long long r = atomicAdd(&P.st->bar, 1ull << 32) >> 32;
            atomicAdd(&P.st->ndef[slot >= P.round_tiles], 1ull);
            if (r < P.rec_cap) {
                P.recs[r].start = (unsigned long long)(a + p);
                P.recs[r].doc = (unsigned long long)dc;  // the document holding the tile's first byte
            }
            S.sid[SI(p)] = 0xFF000000u;
            S.sid[SI(p + 1)] = (uint32_t)r;
            S.n_def = 1;
            continue;
        }
        const uint32_t len = (uint32_t)(e - p);
        if (len == 1) {
            S.sid[SI(p)] = (1u << 24) | C.base[sb_byte(sb, p)];
            continue;
        }
        const uint32_t id = use_memo ? memo_lookup(T, sb, (uint32_t)p, len) : GPUBPE_INF;
        if (id == GPUBPE_INF) {  // not a memoised vocab string: the warp engine below
            S.u.a.miss[atomicAdd(&S.n_miss, 1u)] = (uint32_t)p | (len << 16);
            ++c_miss;
            continue;
        }
        ++c_memo;
        S.sid[SI(p)] = (1u << 24) | id;
    }
    TSTAMP(7, c_seg);
    __syncwarp();
    TSTAMP(2, c_memo);

    // ---- 6. memo misses: packed into the lanes, exact multi-merge passes
    {
        const bool strict = P.strict || !T.well_formed;
        const uint32_t nm = S.n_miss;
#pragma unroll 1
        for (uint32_t i = 0; i < nm;) {
            uint32_t k = 1, tot = S.u.a.miss[i] >> 16;
            if (!strict || GPUBPE_SEQ_ENGINE)  // (the sequential engine is exact for any table)
                while (i + k < nm && tot + (S.u.a.miss[i + k] >> 16) <= 32) tot += S.u.a.miss[i + k++] >> 16;
#ifdef GPUBPE_DEBUG_STAMPS
            long long eng_acc[6] = {0, 0, 0, 0, 0, 0};
            const uint32_t np_ = GPUBPE_SEQ_ENGINE ? warp_seq_bpe(T, C.base, sb, S.sid, S.u.a.miss + i, k, eng_acc)
                                                   : warp_pack_bpe(T, C.base, sb, S.sid, S.u.a.miss + i, k, strict, eng_acc);
            if (P.dbg && lane == 0) {
                for (int q = 0; q < 6; ++q) atomicAdd(&P.dbg[32768 + q], (unsigned long long)eng_acc[q]);
                atomicAdd(&P.dbg[32768 + 6], (unsigned long long)np_);
                atomicAdd(&P.dbg[32768 + 7], 1ull);
            }
            c_pass += np_;
#else
            if (GPUBPE_SEQ_ENGINE) c_pass += warp_seq_bpe(T, C.base, sb, S.sid, S.u.a.miss + i, k);
            else c_pass += warp_pack_bpe(T, C.base, sb, S.sid, S.u.a.miss + i, k, strict);
#endif
            i += k;
        }
    }
    TSTAMP(3, c_pass);
#ifdef GPUBPE_DEBUG_STAMPS
    if (P.dbg && t < 2048 && lane == 0) P.dbg[16384 + 8 * t + 6] = S.n_miss;
#endif

    // ---- 7. entries in output order (chunked scan over the list) -> outbuf;
    //         each segment's sid slot then holds its entry offset (when step 8 runs)
    const bool need_offs = (P.n_docs > 1 || a == 0 || last) && !(inner && !last);
    uint32_t total = 0;
#pragma unroll 1
    for (uint32_t i0 = 0; i0 < nseg; i0 += 32) {
        const uint32_t i = i0 + lane;
        const bool valid = i < nseg;
        const int p = valid ? S.seg[i] : 0;
        const uint32_t v = valid ? S.sid[SI(p)] : 0u;
        const uint32_t cc = valid ? seg_entries(v) : 0u;
        uint32_t incl;
        if (__all_sync(FULL_MASK, cc <= 1u)) {  // one entry per segment (nearly always): no scan
            incl = min((uint32_t)lane + 1u, nseg - i0);  // (the valid lanes are a prefix)
        } else {
            incl = cc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(FULL_MASK, incl, o);
                if (lane >= o) incl += y;
            }
        }
        const uint32_t o = total + incl - cc;
        if (valid) {
            if ((v >> 24) == 0xFFu) {
                S.u.outbuf[o] = MARK | S.sid[SI(p + 1)];
            } else {
                S.u.outbuf[o] = v & 0xFFFFFFu;
#pragma unroll 1
                for (uint32_t j = 1; j < cc; ++j) S.u.outbuf[o + j] = S.sid[SI(p + j)];
            }
            if (need_offs) S.sid[SI(p)] = o;  // (read by step 8 only)
        }
        total += __shfl_sync(FULL_MASK, incl, 31);
    }
    __syncwarp();
    {
        uint4 *dst = reinterpret_cast<uint4 *>(P.scratch + slot * SLOT);
        const uint4 *src = reinterpret_cast<const uint4 *>(S.u.outbuf);
#pragma unroll 1
        for (uint32_t k = lane; k < (total + 3) / 4; k += 32) dst[k] = src[k];
        if (lane == 0) P.tiles[slot] = (unsigned long long)total | ((unsigned long long)S.n_def << 16);
    }
    TSTAMP(4, total);

    // ---- 8. tile-local entry offsets of the documents starting in this tile
    if (need_offs) {
        long long dlb;  // first document with offs >= a
        if (__ldg(&P.doc_offs[dc]) < a) {
            dlb = dc + 1;
        } else {
            dlb = dc;
#pragma unroll 1
            for (;;) {  // empty documents just before dc also start at a
                const long long d = dlb - 1 - lane;
                const bool eq = d >= 0 && __ldg(&P.doc_offs[d]) == a;
                const unsigned m = __ballot_sync(FULL_MASK, eq);
                const int run = m == FULL_MASK ? 32 : __ffs(~m) - 1;
                dlb -= run;
                if (run < 32) break;
            }
        }
#pragma unroll 1
        for (long long d0 = dlb;; d0 += 32) {
            const long long d = d0 + lane;
            bool in = false;
            if (d <= (long long)P.n_docs) {
                const long long s = __ldg(&P.doc_offs[d]);
                if (s < a + nin || last) {
                    in = true;
                    const int q = (int)(s - a);
                    P.out_offs[d] = (long long)(q >= nin ? total : S.sid[SI(q)]);
                }
            }
            if (__ballot_sync(FULL_MASK, in) != FULL_MASK) break;
        }
    }
    __syncwarp();
    TSTAMP(5, 0);
    X.n_segments += c_seg;
    X.memo_hits += c_memo;
    X.short_merges += c_miss;
    if (lane == 0) X.engine_passes += c_pass;
    return total | (S.n_def << 16);
}

// ------------------------------------------------------------------ phase B

// Extra ids of the deferred markers among the first n entries of a slot
// (one thread; only for tiles that hold markers).
__device__ unsigned long long marker_extra(const EncodeParams &P, const uint32_t *src, uint32_t n) {
    unsigned long long x = 0;
    for (uint32_t k = 0; k < n; ++k) {
        const uint32_t e = __ldcg(&src[k]);
        if (e & MARK) x += (unsigned long long)__ldcg(&P.recs[e & ~MARK].count) - 1;
    }
    return x;
}

// Warp: copy one tile's slot to out_ids[base ...], expanding deferred markers.
__device__ void place_tile(const EncodeParams &P, const uint32_t *src, unsigned long long w,
                           unsigned long long base) {
    const int lane = threadIdx.x & 31;
    const DevTables &T = P.T;
    const uint32_t n = TW_ENTRIES(w);
    uint32_t *dst = P.out_ids + base;
    if (!TW_HASDEF(w)) {
        for (uint32_t k = lane; k < n; k += 32) dst[k] = out_id(T, __ldcg(&src[k]));
    } else {
        unsigned long long o = 0;
        for (uint32_t k0 = 0; k0 < n; k0 += 32) {
            const uint32_t k = k0 + lane;
            const uint32_t e = k < n ? __ldcg(&src[k]) : 0u;
            const bool mark = k < n && (e & MARK);
            uint32_t cntk = 0, res = 0;
            if (mark) {
                cntk = __ldcg(&P.recs[e & ~MARK].count);
                res = __ldcg(&P.recs[e & ~MARK].res);
            } else if (k < n) {
                cntk = 1;
            }
            unsigned long long incl = cntk;
#pragma unroll
            for (int s = 1; s < 32; s <<= 1) {
                const unsigned long long y = __shfl_up_sync(FULL_MASK, incl, s);
                if (lane >= s) incl += y;
            }
            const unsigned long long ex = o + incl - cntk;
            if (k < n && !mark) dst[ex] = out_id(T, e);
            for (unsigned mk = __ballot_sync(FULL_MASK, mark); mk; mk &= mk - 1) {
                const int src_lane = __ffs(mk) - 1;
                const unsigned long long at = __shfl_sync(FULL_MASK, ex, src_lane);
                const uint32_t c = __shfl_sync(FULL_MASK, cntk, src_lane);
                const uint32_t r = __shfl_sync(FULL_MASK, res, src_lane);
                if (c >= GIANT_MIN - 1) {  // a giant's ids: copied by the whole grid after placement
                    const uint32_t rec = __shfl_sync(FULL_MASK, e & ~MARK, src_lane);
                    if (lane == 0) P.recs[rec].dst = base + at;
                    continue;
                }
                for (uint32_t j = lane; j < c; j += 32) dst[at + j] = out_id(T, __ldcg(&P.arena[r + j]));
            }
            o += __shfl_sync(FULL_MASK, incl, 31);
        }
    }
    __syncwarp();
    // the slot is dead: drop its lines from L2 without write-back (tiles with
    // markers are re-read by the document fix-up)
    if (!TW_HASDEF(w))
        for (uint32_t k = lane; k < (n * 4 + 127) / 128; k += 32) l2_discard(src + 32 * k);
}

// CSR offsets of the documents starting in tiles [lo, hi) (C.tw / C.tb hold
// their words and in-range offsets): tile-local -> global.
__device__ __forceinline__ void fix_doc_offsets(const EncodeParams &P, CtaSmem &C, unsigned long long lo,
                                                unsigned long long hi, int nt, unsigned long long base,
                                                const uint32_t *slots) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    // One document: its offsets are 0 and the id total, no look-ups needed.
    if (P.n_docs == 1) {
        if (tid == 0 && nt > 0) {
            if (lo == 0) P.out_offs[0] = 0;
            if (hi == P.n_tiles) P.out_offs[1] = (long long)(base + C.bcast[2]);
        }
    } else if (wid == 0 && nt > 0) {
        const long long blo = (long long)lo * P.tile_bytes;
        long long d = 0;
        if (blo > 0) {  // first document with offs >= blo (lower bound)
            long long lo_d = 0, hi_d = (long long)P.n_docs;  // answer in [lo_d, hi_d]
            while (hi_d > lo_d) {
                const long long step = (hi_d - lo_d + 31) / 32;
                const long long idx = lo_d + (long long)lane * step;
                const bool lt = idx < hi_d && __ldg(&P.doc_offs[idx]) < blo;
                const unsigned m = __ballot_sync(FULL_MASK, lt);
                if (!m) { hi_d = lo_d; break; }
                const int l = 31 - __clz(m);
                lo_d = lo_d + (long long)l * step + 1;
                hi_d = min(hi_d, lo_d - 1 + step);
            }
            d = lo_d;
        }
        for (long long d0 = d;; d0 += 32) {
            const long long dd = d0 + lane;
            bool in = false;
            if (dd <= (long long)P.n_docs) {
                const long long s = __ldg(&P.doc_offs[dd]);
                if (s < (long long)hi * P.tile_bytes || hi == P.n_tiles) in = s >= blo;
                if (in) {
                    const long long t = min(s >> (31 - __clz(P.tile_bytes)), (long long)P.n_tiles - 1);  // wt: 2^k
                    const int k = (int)(t - (long long)lo);
                    const uint32_t local = (uint32_t)__ldcg(&P.out_offs[dd]);
                    unsigned long long v = base + C.tb[k] + local;
                    if (TW_HASDEF(C.tw[k])) v += marker_extra(P, slots + (size_t)k * SLOT, local);
                    P.out_offs[dd] = (long long)v;
                }
            }
            if (__ballot_sync(FULL_MASK, in) != FULL_MASK) break;
        }
    }
}

// CTA: place the tiles [lo, hi) of round r (unit u = r * grid + blockIdx.x).
__device__ __noinline__ void place_range(const EncodeParams &P, CtaSmem &C, unsigned long long r,
                            unsigned long long t0, unsigned long long lo, unsigned long long hi) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const unsigned long long par = r & 1;
    const unsigned long long *tw = P.tiles + par * P.round_tiles + (lo - t0);
    const uint32_t *slots = P.scratch + (par * P.round_tiles + (lo - t0)) * SLOT;
    const int nt = (int)(hi - lo);
    const unsigned long long u = r * gridDim.x + blockIdx.x;
    // A call that fits one round needs no look-back: warps 1.. sum the words
    // of all tiles before this range directly (L2 reads, no CTA waits on
    // another) while warp 0 scans the range.
    const bool direct = r == 0 && P.n_tiles <= P.round_tiles;
    if (direct && wid > 0) {
        unsigned long long acc = 0;
        for (unsigned long long t = (unsigned long long)(tid - 32); t < lo; t += NT - 32) {
            const unsigned long long w = __ldcg(&P.tiles[t]);  // round 0: parity 0, t0 == 0
            acc += TW_ENTRIES(w) + TW_EXTRA(w);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL_MASK, acc, o);
        if (lane == 0) C.red[wid][0] = acc;
    }
    if (wid == 0) {
        constexpr int PER = UNIT_MAX / 32;
        unsigned long long v[PER], sum = 0;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int k = lane * PER + j;
            unsigned long long w = k < nt ? __ldcg(&tw[k]) : 0ull;
            C.tw[k] = w;
            v[j] = TW_ENTRIES(w) + TW_EXTRA(w);
            sum += v[j];
        }
        unsigned long long incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(FULL_MASK, incl, o);
            if (lane >= o) incl += y;
        }
        const unsigned long long total = __shfl_sync(FULL_MASK, incl, 31);
        unsigned long long o = incl - sum;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            C.tb[lane * PER + j] = o;
            o += v[j];
        }
        unsigned long long base = 0;
        if (direct) {
            // base comes from warps 1.. (C.bcast[1]) after the barrier below
        } else if (nt > 0) {
            base = warp_lookback(P.status, u, total, P.epoch);
        } else if (lane == 0) {  // empty unit: an aggregate of 0 keeps the chain moving
            st_relaxed(&P.status[u], ((unsigned long long)P.epoch << 44) | (LB_AGG << 42));
        }
        if (lane == 0) {
            C.bcast[0] = base;
            C.bcast[2] = total;
        }
    }
    __syncthreads();
    unsigned long long base = C.bcast[0];
    if (direct) {  // every warp sums the partials of warps 1..
        base = lane > 0 && lane < NW ? C.red[lane][0] : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) base += __shfl_xor_sync(FULL_MASK, base, o);
    }
    if (tid == 0 && nt > 0 && hi == P.n_tiles) P.st->n_ids = base + C.bcast[2];
    if (P.dbg && tid == 0 && r == 0) P.dbg[36864 + 4 * blockIdx.x + 1] = gtimer();
    for (int k = wid; k < nt; k += NW) place_tile(P, slots + (size_t)k * SLOT, C.tw[k], base + C.tb[k]);
    if (P.dbg && lane == 0 && r == 0) atomicMax(&P.dbg[36864 + 4 * blockIdx.x + 2], gtimer());
    fix_doc_offsets(P, C, lo, hi, nt, base, slots);
    __syncthreads();
}

// All CTAs (co-resident: cooperative launch).  k = 1, 2, ... per use.
// Grid barrier k (1, 2, ...).  *defs (shared memory, optional) receives the
// deferred-segment count, final once every CTA has arrived.
__device__ void grid_sync(EncodeState *st, unsigned int k, unsigned long long *defs = nullptr) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(&st->bar, 1ull);
        const unsigned long long target = (unsigned long long)k * gridDim.x;
        unsigned long long w;
        while (((w = ld_relaxed(&st->bar)) & 0xFFFFFFFFull) < target) __nanosleep(128);
        __threadfence();  // acquire side of the barrier, once
        if (defs) *defs = w >> 32;
    }
    __syncthreads();
}

#ifndef GPUBPE_POLL_NS
#define GPUBPE_POLL_NS 256
#endif
// One-round calls: wait until every tile of the call is done -- per placement
// range one word (tiles done << 40 | entries), one release add per tile --
// then C.bcast[0] = the entries of the ranges before this CTA's and
// C.bcast[3] = the deferred segments recorded (final once every tile is done).
// This replaces the grid barrier and the prefix over every tile word.
__device__ void complete_one_round(const EncodeParams &P, CtaSmem &C, unsigned long long q) {
    if ((threadIdx.x >> 5) == 0) {
        const int lane = threadIdx.x & 31;
        const unsigned long long G = gridDim.x, n = P.n_tiles;
        unsigned long long before;
        for (;;) {
            bool ok = true;
            before = 0;
#pragma unroll
            for (int k = 0; k < RNG_MAX / 32; ++k) {
                const unsigned long long j = (unsigned long long)(lane + 32 * k);
                if (j < G) {
                    const unsigned long long v = ld_relaxed(&P.st->rng[j]);
                    const unsigned long long l = j * q, h = min(n, l + q);
                    ok &= (v >> 40) == (h > l ? h - l : 0ull);
                    if (j < blockIdx.x) before += v & ((1ull << 40) - 1);
                }
            }
            if (__all_sync(FULL_MASK, ok)) break;
            __nanosleep(GPUBPE_POLL_NS);  // (the poller shares its SM with the slowest tiles' warps)
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) before += __shfl_xor_sync(FULL_MASK, before, o);
        if (lane == 0) {
            __threadfence();  // acquire: the tiles' slots, words and records
            C.bcast[0] = before;
            C.bcast[3] = ld_relaxed(&P.st->ndef[0]);
        }
    }
    __syncthreads();
}

// One-round calls without deferred segments: CTA c places its range [lo, hi)
// of at most NW tiles.  Every warp loads the range's tile words (one per lane)
// and, speculatively and in the same round trip, the first entries of its own
// tile's slot; base = entries of the ranges before (complete_one_round).
__device__ __noinline__ void place_range_one(const EncodeParams &P, CtaSmem &C, unsigned long long lo,
                                             unsigned long long hi, unsigned long long base) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int nt = (int)(hi - lo);
    if (P.dbg && tid == 0) P.dbg[38000 + 4 * blockIdx.x] = gtimer();
    const uint32_t *slots = P.scratch + lo * SLOT;  // round 0: parity 0, t0 = 0
    const uint32_t *src = slots + (size_t)wid * SLOT;
    constexpr int PRE = 5;  // entries per lane fetched before the count is known (wt 128: <= 160)
    uint32_t pre[PRE];
    const unsigned long long w = lane < nt ? __ldcg(&P.tiles[lo + lane]) : 0ull;
    if (wid < nt) {
#pragma unroll
        for (int j = 0; j < PRE; ++j) pre[j] = __ldcg(&src[lane + 32 * j]);
    }
    const uint32_t e = TW_ENTRIES(w);
    if (P.dbg && lane == 0) atomicMax(&P.dbg[38000 + 4 * blockIdx.x + 1], gtimer() + (e & 0));
    uint32_t incl = e;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL_MASK, incl, o);
        if (lane >= o) incl += y;
    }
    const uint32_t excl = incl - e;
    if (wid == 0) {
        C.tw[lane] = w;
        C.tb[lane] = excl;
        if (lane == 31) C.bcast[2] = incl;
    }
    if (wid < nt) {
        const uint32_t n = __shfl_sync(FULL_MASK, e, wid);
        const uint32_t off = __shfl_sync(FULL_MASK, excl, wid);
        uint32_t *dst = P.out_ids + base + off;
#pragma unroll
        for (int j = 0; j < PRE; ++j) {
            const uint32_t k = lane + 32 * j;
            if (k < n) dst[k] = out_id(P.T, pre[j]);
        }
        for (uint32_t k = lane + 32 * PRE; k < n; k += 32) dst[k] = out_id(P.T, __ldcg(&src[k]));
        if (P.dbg && lane == 0) atomicMax(&P.dbg[36864 + 4 * blockIdx.x + 0], gtimer());
        // (no L2 discard of the slot here: one discard per line costs ~1 us at the
        // tail of a latency-bound call; these few MB are written back later)
        if (P.dbg && lane == 0) atomicMax(&P.dbg[36864 + 4 * blockIdx.x + 2], gtimer());
    }
    __syncthreads();
    if (tid == 0 && hi == P.n_tiles) P.st->n_ids = base + C.bcast[2];
    fix_doc_offsets(P, C, lo, hi, nt, base, slots);
}

// Warp: its lanes' counters summed into C.red[wid] (part 1 of publish_counters).
__device__ __forceinline__ void warp_counters(CtaSmem &C, const WarpCtx &X) {
    const int lane = threadIdx.x & 31;
    unsigned long long seg = X.n_segments, memo = X.memo_hits, sm = X.short_merges, ep = X.engine_passes;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        seg += __shfl_xor_sync(FULL_MASK, seg, o);
        memo += __shfl_xor_sync(FULL_MASK, memo, o);
        sm += __shfl_xor_sync(FULL_MASK, sm, o);
        ep += __shfl_xor_sync(FULL_MASK, ep, o);
    }
    const int wid = threadIdx.x >> 5;
    if (lane == 0) {
        C.red[wid][0] = seg;
        C.red[wid][1] = memo;
        C.red[wid][2] = sm;
        C.red[wid][3] = ep;
    }
}

// One warp, after a CTA barrier that follows every warp's warp_counters: the
// CTA's sums, then one global add per counter (part 2).
__device__ __forceinline__ void cta_counters(CtaSmem &C, PassCounters *dst) {
    const int lane = threadIdx.x & 31;
    unsigned long long v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        v[q] = lane < NW ? C.red[lane][q] : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(FULL_MASK, v[q], o);
    }
    if (lane == 0) {
        C.pc.n_segments += v[0];
        C.pc.memo_hits += v[1];
        C.pc.short_merges += v[2];
        C.pc.engine_passes += v[3];
        const unsigned long long *s = &C.pc.n_segments;
        unsigned long long *d = &dst->n_segments;
        for (int i = 0; i < (int)(sizeof(PassCounters) / 8); ++i)
            if (s[i]) atomicAdd(&d[i], s[i]);
    }
}

// Sum the warps' counters into the CTA, then into the call's global set.
__device__ void publish_counters(CtaSmem &C, WarpCtx &X, PassCounters *dst) {
    warp_counters(C, X);
    __syncthreads();
    if ((threadIdx.x >> 5) == 0) cta_counters(C, dst);
}

#define REC_GIANT 0xFFFFFFFFu  // record marked by the warp pass: a whole-grid job

// ------------------------------------------------------------------ grid engine
//
// Exact multi-merge BPE of ONE giant segment by all CTAs (engine.cuh's
// selection rule, same arena layout).  CTA c owns elements [c*n/G, (c+1)*n/G)
// of the current sequence; a pass costs three grid barriers:
//   A  block min (rank, pos) -> atomicMin; last run start of the range -> gscr;
//   B  selection with the run-start carry of the ranges before; the pair just
//      before the range is re-selected redundantly (same inputs, same rule),
//      so keep counts need no extra barrier; counts -> gscr;
//   C  compaction at the global prefix of the counts (neighbours' selections
//      were written before barrier B).
// Strict passes add two barriers (B0: candidates marked, then the first one
// whose merge creates a pair of rank <= r_min, engine.cuh strict_violates).
// gscr: [0], [1] alternating kmin slots, [2] giant end, [3] arena offset,
// [5], [6] alternating strict first-violation slots,
// [8 + c] last run start + 1 of range c, [8 + G + c] kept tokens of range c.

__device__ __forceinline__ bool grid_select(const DevTables &T, const EngineMem &M, uint32_t i, uint32_t n,
                                            uint32_t s, uint32_t rmin, uint32_t pmin, bool strict,
                                            unsigned long long vfirst) {
    if (i + 1 >= n) return false;
    const uint32_t r = M.pr[i].x;
    if (strict) return STRICT_MULTI ? __ldcg(&M.sel[i]) && i <= vfirst : i == pmin;  // (marks of B0)
    bool ok = r != GPUBPE_INF && ((i - s) & 1u) == 0;
    if (ok && r != rmin) ok = walk_left(T, M.tok, M.pr, s, r) && walk_right(T, M.tok, M.pr, i + 1, n, r);
    return ok;
}

__device__ uint32_t grid_engine_run(const EncodeParams &P, CtaSmem &C, EngineMem M, uint32_t n, bool strict,
                                    unsigned int &nbar, uint32_t *passes_out, const uint32_t **out) {
    const uint32_t tid = threadIdx.x, G = gridDim.x, c = blockIdx.x;
    const DevTables &T = P.T;
    EncodeState *st = P.st;
    unsigned long long *g = P.gscr;
    for (unsigned long long i = (unsigned long long)c * NT + tid; i + 1 < n; i += (unsigned long long)G * NT) {
        const PairHit h = probe_pair(T, M.tok[i], M.tok[i + 1]);
        M.pr[i] = make_uint2(h.rank, h.nw);
    }
    if (c == 0 && tid == 0) g[0] = g[1] = g[5] = g[6] = ~0ull;
    grid_sync(st, ++nbar);
    uint32_t passes = 0;
    while (n >= 2) {
        const uint32_t lo = (uint32_t)((unsigned long long)n * c / G), hi = (uint32_t)((unsigned long long)n * (c + 1) / G);
        // ---- A: min and the range's last run start
        unsigned long long mine = ~0ull;
        uint32_t ls = 0;  // last start + 1 (0: none)
        for (uint32_t i = lo + tid; i < hi; i += NT) {
            if (i + 1 < n) {
                const uint32_t r = M.pr[i].x;
                if (r != GPUBPE_INF) mine = min(mine, ((unsigned long long)r << 32) | i);
                if (i == 0 || M.pr[i - 1].x != r) ls = i + 1;
            }
        }
        const unsigned long long bmin = block_min_u64(mine, C.es);
        uint32_t dummy;
        const uint32_t bls = block_incl_max(ls, C.es, &dummy);
        if (tid == NT - 1) {
            if (bmin != ~0ull) atomicMin(&g[passes & 1], bmin);
            g[8 + c] = bls;  // inclusive max of the last thread = the range's last start + 1
        }
        grid_sync(st, ++nbar);
        if (c == 0 && tid == 0) g[(passes + 1) & 1] = ~0ull;  // the next pass's slot
        const unsigned long long kmin = __ldcg(&g[passes & 1]);
        if (kmin == ~0ull) break;  // (every CTA sees the same value)
        const uint32_t rmin = (uint32_t)(kmin >> 32), pmin = (uint32_t)kmin;
        // carry: last run start before this range
        uint32_t carry = 0;
        for (uint32_t q = tid; q < c; q += NT) carry = max(carry, (uint32_t)__ldcg(&g[8 + q]));
        carry = block_incl_max(carry, C.es, &dummy);
        if (tid == 0) C.bcast[1] = dummy;
        __syncthreads();
        carry = (uint32_t)C.bcast[1];
        const uint32_t s_before = carry ? carry - 1 : 0u;  // run start covering lo - 1
        // ---- B0 (strict): candidates marked in M.sel, then the first one whose merge
        //      creates a pair of rank <= r_min (engine.cuh strict_violates), grid-wide;
        //      two barriers more
        unsigned long long vfirst = ~0ull;
        if (strict && STRICT_MULTI) {
            uint32_t runs = carry;
            for (uint32_t b = lo; b < hi; b += NT) {
                const uint32_t i = b + tid;
                const bool pair = i < hi && i + 1 < n;
                const uint32_t r = pair ? M.pr[i].x : GPUBPE_INF;
                const bool start = pair && (i == 0 || M.pr[i - 1].x != r);
                uint32_t chunk_max;
                uint32_t sv = block_incl_max(start ? i + 1 : 0u, C.es, &chunk_max);
                sv = max(sv, runs);
                runs = max(runs, chunk_max);
                if (i < hi) M.sel[i] = pair && r == rmin && ((i - (sv ? sv - 1 : 0u)) & 1u) == 0;
            }
            grid_sync(st, ++nbar);
            unsigned long long first = ~0ull;
            for (uint32_t i = lo + tid; i < hi; i += NT)
                if (__ldcg(&M.sel[i]) && strict_violates(T, M, i, n, rmin)) first = min(first, (unsigned long long)i);
            const unsigned long long bf = block_min_u64(first, C.es);
            if (tid == 0 && bf != ~0ull) atomicMin(&g[5 + (passes & 1)], bf);
            grid_sync(st, ++nbar);
            if (c == 0 && tid == 0) g[5 + ((passes + 1) & 1)] = ~0ull;  // the next pass's slot
            vfirst = __ldcg(&g[5 + (passes & 1)]);
        }
        // ---- B: selection of [lo, hi), redundant selection of lo - 1, keep counts
        const bool sel_prev = lo > 0 && grid_select(T, M, lo - 1, n, s_before, rmin, pmin, strict, vfirst);
        uint32_t runs = carry;  // max start + 1 seen so far
        for (uint32_t b = lo; b < hi; b += NT) {
            const uint32_t i = b + tid;
            const bool pair = i < hi && i + 1 < n;
            const uint32_t r = pair ? M.pr[i].x : GPUBPE_INF;
            const bool start = pair && (i == 0 || M.pr[i - 1].x != r);
            uint32_t chunk_max;
            uint32_t sv = block_incl_max(start ? i + 1 : 0u, C.es, &chunk_max);
            sv = max(sv, runs);
            runs = max(runs, chunk_max);
            if (i < hi) {
                if (strict) {
                    M.sel[i] = grid_select(T, M, i, n, sv ? sv - 1 : 0u, rmin, pmin, strict, vfirst);
                } else {  // walks deferred to the loop below (no barrier between the walks)
                    const uint32_t s = sv ? sv - 1 : 0u;
                    const bool ok = pair && r != GPUBPE_INF && ((i - s) & 1u) == 0;
                    M.sel[i] = ok;
                    M.tok2[i] = ok && r != rmin ? s : GPUBPE_INF;  // (tok2 is free until phase C)
                }
            }
        }
        if (!strict)  // the same positions per thread as above
            for (uint32_t i = lo + tid; i < hi; i += NT) {
                const uint32_t s = M.tok2[i];
                if (s != GPUBPE_INF) {
                    const uint32_t r = M.pr[i].x;
                    M.sel[i] = walk_left(T, M.tok, M.pr, s, r) && walk_right(T, M.tok, M.pr, i + 1, n, r);
                }
            }
        __syncthreads();
        uint32_t kept = 0;
        for (uint32_t j = lo + tid; j < hi; j += NT) {
            const bool sp = j == lo ? sel_prev : (M.sel[j - 1] != 0);
            kept += (j > 0 && sp) ? 0u : 1u;
        }
        uint32_t ktot;
        (void)block_excl_sum(kept, C.es, &ktot);
        if (tid == 0) g[8 + G + c] = ktot;
        grid_sync(st, ++nbar);
        // ---- C: compaction at the global prefix
        uint32_t pre = 0, tot = 0;
        for (uint32_t q = tid; q < G; q += NT) {
            const uint32_t v = (uint32_t)__ldcg(&g[8 + G + q]);
            tot += v;
            if (q < c) pre += v;
        }
        uint32_t ptot;
        pre = block_excl_sum(pre, C.es, &ptot);  // (sum over threads)
        pre = ptot;
        (void)block_excl_sum(tot, C.es, &tot);
        uint32_t carry2 = pre;
        for (uint32_t b = lo; b < hi; b += NT) {
            const uint32_t j = b + tid;
            bool keep = false;
            if (j < hi) {
                const bool sp = j == lo ? sel_prev : (__ldcg(&M.sel[j - 1]) != 0);
                keep = !(j > 0 && sp);
            }
            uint32_t total;
            const uint32_t pos = carry2 + block_excl_sum(keep ? 1u : 0u, C.es, &total);
            carry2 += total;
            if (keep) {
                const bool sj = __ldcg(&M.sel[j]) != 0;
                const uint2 pj = (j + 1 < n) ? M.pr[j] : make_uint2(GPUBPE_INF, 0);
                const uint32_t t = sj ? pj.y : M.tok[j];
                M.tok2[pos] = t;
                const uint32_t jn = sj ? j + 2 : j + 1;
                if (jn < n) {
                    const bool sn = __ldcg(&M.sel[jn]) != 0;
                    if (sj || sn) {
                        if (pos + 1 == pre + ktot) {  // the range's last pair: its right token is the next range's
                            const uint32_t tn = sn ? M.pr[jn].y : M.tok[jn];
                            const PairHit h = probe_pair(T, t, tn);
                            M.pr2[pos] = make_uint2(h.rank, h.nw);
                        } else {
                            M.pr2[pos] = make_uint2(GPUBPE_INF, REPROBE);  // probed below
                        }
                    } else {
                        M.pr2[pos] = pj;
                    }
                }
            }
        }
        __syncthreads();
        // re-probes inside the range's output (no barrier between the probes)
        for (uint32_t p = pre + tid; p + 1 < pre + ktot; p += NT) {
            const uint2 v = M.pr2[p];
            if (v.x == GPUBPE_INF && v.y == REPROBE) {
                const PairHit h = probe_pair(T, M.tok2[p], M.tok2[p + 1]);
                M.pr2[p] = make_uint2(h.rank, h.nw);
            }
        }
        grid_sync(st, ++nbar);
        n = tot;
        uint32_t *tt = M.tok; M.tok = M.tok2; M.tok2 = tt;
        uint2 *pp = M.pr; M.pr = M.pr2; M.pr2 = pp;
        ++passes;
    }
    *passes_out = passes;
    *out = M.tok;
    return n;
}

// Giant-list entries [gi0, gi0 + NT) whose record passes `test`, as one bit
// mask per warp in gmask(C): every thread loads one entry, so the list is
// scanned at the width of the CTA instead of one dependent pair of L2 loads
// per entry (1,000 giants in a call: ~2,000 round trips per scan before).
// (the masks live in C.tb: placement scratch, dead while giants are encoded
// and after the placement's closing barrier)
__device__ __forceinline__ uint32_t *gmask(CtaSmem &C) { return reinterpret_cast<uint32_t *>(C.tb); }
static_assert(UNIT_MAX * 2 >= NW, "giant masks alias C.tb");
template <class F>
__device__ __forceinline__ void giant_masks(const EncodeParams &P, CtaSmem &C, unsigned long long gi0,
                                            unsigned long long ng, F test) {
    __syncthreads();  // the previous window's masks are read
    const unsigned long long gi = gi0 + threadIdx.x;
    const bool hit = gi < ng && test(&P.recs[__ldcg(&P.glist[gi])]);
    const uint32_t m = __ballot_sync(FULL_MASK, hit);
    if ((threadIdx.x & 31) == 0) gmask(C)[threadIdx.x >> 5] = m;
    __syncthreads();
}

// All CTAs: encode the giant records of [d0, d1) one after another.
__device__ void grid_giants(const EncodeParams &P, CtaSmem &C, unsigned long long t0, unsigned long long par,
                            unsigned int &nbar, long long mmax) {
    const int tid = threadIdx.x;
    EncodeState *st = P.st;
    unsigned long long *g = P.gscr;
    const long long N = (long long)P.n_bytes;
    const bool strict = P.strict || !P.T.well_formed;
    const unsigned long long ng = __ldcg(&g[4]);  // giants of this round (same in every CTA)
    // (records without the mark were encoded by one CTA, cta_giants)
    for (unsigned long long gi0 = 0; gi0 < ng; gi0 += NT) {
      giant_masks(P, C, gi0, ng, [](const DefRec *rec) { return __ldcg(&rec->count) == REC_GIANT; });
      for (int w = 0; w < NW; ++w)
      for (uint32_t m = gmask(C)[w]; m; m &= m - 1) {
        const unsigned long long gi = gi0 + 32 * w + (__ffs(m) - 1);
        const unsigned long long r = __ldcg(&P.glist[gi]);
        const long long s0 = (long long)__ldcg(&P.recs[r].start);
        // the segment's end: each CTA scans a slice of [s0 + mmax + 1, lim)
        long long d = 0;
        if (P.n_docs > 1) {
            if ((threadIdx.x >> 5) == 0) {
                const long long dd = warp_doc_from(P.doc_offs, (long long)__ldcg(&P.recs[r].doc), P.n_docs, s0);
                if ((threadIdx.x & 31) == 0) C.bcast[1] = (unsigned long long)dd;
            }
            __syncthreads();
            d = (long long)C.bcast[1];
        }
        long long lim = next_struct_cut(P, d, s0);
        if (lim > N) lim = N;
        const long long from = s0 + mmax + 1, span = lim - from;
        const long long lo = from + span * blockIdx.x / gridDim.x, hi = from + span * (blockIdx.x + 1) / gridDim.x;
        if (blockIdx.x == 0 && tid == 0) g[2] = (unsigned long long)lim;
        grid_sync(st, ++nbar);
        const long long e = cta_first_nonjunction(P, C.jb, lo, hi, C.es);
        if (tid == 0 && e < hi) atomicMin(&g[2], (unsigned long long)e);
        if (blockIdx.x == 0 && tid == 0) {
            // arena for the engine (the length is not known yet: bound it by lim)
            const unsigned long long words = (ENGINE_BYTES(lim - s0) + 15) / 16 * 4;
            unsigned long long off = atomicAdd(&st->arena_used, words);
            if (off + words > P.arena_words) {
                atomicExch(&st->overflow, 1ull);
                off = ~0ull;
            }
            g[3] = off;
        }
        grid_sync(st, ++nbar);
        const unsigned long long off = __ldcg(&g[3]);
        const long long send = (long long)__ldcg(&g[2]);
        if (off == ~0ull) continue;  // the host re-runs with a larger arena (all CTAs alike)
        const unsigned long long len = (unsigned long long)(send - s0);
        EngineMem M;
        M.tok = P.arena + off;
        M.tok2 = M.tok + len;
        M.pr = reinterpret_cast<uint2 *>(M.tok2 + len);
        M.pr2 = M.pr + len;
        M.sel = reinterpret_cast<uint8_t *>(M.pr2 + len);
        for (unsigned long long j = (unsigned long long)blockIdx.x * NT + tid; j < len;
             j += (unsigned long long)gridDim.x * NT)
            M.tok[j] = C.base[__ldg(&P.bytes[s0 + j])];
        grid_sync(st, ++nbar);
        uint32_t passes;
        const uint32_t *res;
        const uint32_t cnt = grid_engine_run(P, C, M, (uint32_t)len, strict, nbar, &passes, &res);
        if (blockIdx.x == 0 && tid == 0) {
            P.recs[r].count = cnt;
            P.recs[r].res = (uint32_t)(res - P.arena);
            const unsigned long long t = (unsigned long long)s0 / (unsigned long long)P.tile_bytes;
            atomicAdd(&P.tiles[par * P.round_tiles + (t - t0)], ((unsigned long long)cnt - 1) << 17);
            atomicAdd(&C.pc.giant_segments, 1ull);
            atomicAdd(&C.pc.giant_bytes, len);
            atomicAdd(&C.pc.engine_passes, (unsigned long long)passes);
        }
      }
    }
}

// Warp: first p in [lo, hi) whose cut slot is a junction miss, else hi.
__device__ long long warp_first_nonjunction(const EncodeParams &P, const uint32_t *jb, long long lo, long long hi) {
    const int lane = threadIdx.x & 31;
    for (long long b = lo; b < hi; b += 16 * 32) {
        const long long p0 = b + 16 * (long long)lane;
        long long k = hi;
        if (p0 < hi) {
            uint32_t x = __ldg(&P.bytes[p0 - 1]);
            const long long pe = min(p0 + 16, hi);
            for (long long p = p0; p < pe; ++p) {
                const uint32_t y = __ldg(&P.bytes[p]);
                const uint32_t idx = (x << 8) | y;
                if (!((jb[idx >> 5] >> (idx & 31)) & 1u) || pretok_cut(P, p)) { k = p; break; }
                x = y;
            }
        }
        const unsigned m = __ballot_sync(FULL_MASK, k < hi);
        if (m) return __shfl_sync(FULL_MASK, k, __ffs(m) - 1);
    }
    return hi;
}

// Group-engine encode of one deferred segment [s0, s0 + len) into the arena;
// the record gets its count and result offset, its tile word the extra ids.
// When the engine's buffers fit `smem` (the group's dead tile staging: the
// round's tiles are done when deferred segments run), the passes run in shared
// memory and only the result goes to the arena (every pass reads and writes
// its whole sequence a few times, each access an L2 round trip in the arena).
#ifndef GPUBPE_SMEM_ENGINE
#define GPUBPE_SMEM_ENGINE 1
#endif
template <class G>
__device__ void encode_record(const EncodeParams &P, CtaSmem &C, const G &g, unsigned long long r, long long s0,
                              unsigned long long len, unsigned long long t0, unsigned long long par, bool lead,
                              unsigned long long *arena_off_bcast, uint32_t *smem, size_t smem_bytes) {
    EncodeState *st = P.st;
    const bool in_smem = GPUBPE_SMEM_ENGINE && ENGINE_BYTES(len) <= smem_bytes;
    if (lead) {
        const unsigned long long words = in_smem ? (len + 3) / 4 * 4 : (ENGINE_BYTES(len) + 15) / 16 * 4;
        unsigned long long off = atomicAdd(&st->arena_used, words);
        if (off + words > P.arena_words) {
            atomicExch(&st->overflow, 1ull);
            off = ~0ull;
        }
        *arena_off_bcast = off;
    }
    g.sync();
    const unsigned long long off = *arena_off_bcast;
    if (off == ~0ull) return;  // the host re-runs with a larger arena
    EngineMem M;
    M.tok = in_smem ? smem : P.arena + off;
    M.tok2 = M.tok + len;
    M.pr = reinterpret_cast<uint2 *>(M.tok2 + len);
    M.pr2 = M.pr + len;
    M.sel = reinterpret_cast<uint8_t *>(M.pr2 + len);
    for (unsigned long long j = g.rank(); j < len; j += g.size()) M.tok[j] = C.base[__ldg(&P.bytes[s0 + j])];
    g.sync();
    uint32_t passes;
    const uint32_t *res;
    const bool strict = P.strict || !P.T.well_formed;
    const uint32_t cnt = engine_run_g(P.T, M, (uint32_t)len, strict, g, &passes, &res);
    if (in_smem) {
        for (uint32_t j = g.rank(); j < cnt; j += g.size()) P.arena[off + j] = res[j];
        res = P.arena + off;
    }
    if (lead) {
        P.recs[r].count = cnt;
        P.recs[r].res = (uint32_t)(res - P.arena);
        const unsigned long long t = (unsigned long long)s0 / (unsigned long long)P.tile_bytes;
        atomicAdd(&P.tiles[par * P.round_tiles + (t - t0)], ((unsigned long long)cnt - 1) << 17);
        if (len >= GIANT_MIN) {
            atomicAdd(&C.pc.giant_segments, 1ull);
            atomicAdd(&C.pc.giant_bytes, len);
        } else {
            atomicAdd(&C.pc.medium_segments, 1ull);
        }
        atomicAdd(&C.pc.engine_passes, (unsigned long long)passes);
    }
    g.sync();
}


// Several giants in a round: each CTA takes giants from the round's list and
// encodes those of at most max_len bytes alone (the block engine, in shared
// memory when it fits), concurrently; longer ones keep their REC_GIANT mark
// for the whole grid (grid_giants).  A lone giant longer than
// GPUBPE_LONE_CTA_MAX is faster on the grid.
__device__ void cta_giants(const EncodeParams &P, CtaSmem &C, unsigned long long t0, unsigned long long par,
                           long long max_len, long long mmax) {
    const int tid = threadIdx.x;
    EncodeState *st = P.st;
    const long long N = (long long)P.n_bytes;
    const unsigned long long ng = __ldcg(&P.gscr[4]);
    for (;;) {
        if (tid == 0) C.bcast[1] = atomicAdd(&st->rec_ctr2, 1ull);
        __syncthreads();
        const unsigned long long gi = C.bcast[1];
        __syncthreads();
        if (gi >= ng) break;
        const unsigned long long r = __ldcg(&P.glist[gi]);
        const long long s0 = (long long)__ldcg(&P.recs[r].start);
        long long d = 0;
        if (P.n_docs > 1) {
            if ((tid >> 5) == 0) {
                const long long dd = warp_doc_from(P.doc_offs, (long long)__ldcg(&P.recs[r].doc), P.n_docs, s0);
                if ((tid & 31) == 0) C.bcast[1] = (unsigned long long)dd;
            }
            __syncthreads();
            d = (long long)C.bcast[1];
            __syncthreads();
        }
        long long lim = next_struct_cut(P, d, s0);
        if (lim > N) lim = N;
        const long long hi = min(lim, s0 + max_len + 1);
        const long long e = cta_first_nonjunction(P, C.jb, s0 + mmax + 1, hi, C.es);
        if (e >= hi && hi < lim) continue;  // longer than max_len: the grid's
        encode_record(P, C, BlockGroup{C.es}, r, s0, (unsigned long long)(e - s0), t0, par, tid == 0, &C.bcast[2],
                      reinterpret_cast<uint32_t *>(C.w), sizeof(C.w));
    }
}

#ifndef GPUBPE_LONE_CTA_MAX
#define GPUBPE_LONE_CTA_MAX 4096
#endif
// Deferred records [d0, d1) of round r.  Pass 1: every warp takes records,
// finds each segment's end (first cut after its start, looked for within
// MEDIUM_MAX + 1 bytes) and encodes the medium ones with the warp engine; longer
// ones are marked.  Pass 2 (after a grid barrier): whole CTAs take the marked
// giants.  Both write results to the arena and extra ids to the tile words.
__device__ __noinline__ void encode_deferred(const EncodeParams &P, CtaSmem &C, unsigned long long d0,
                                             unsigned long long d1, unsigned long long t0, unsigned long long par,
                                             unsigned int &nbar) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    EncodeState *st = P.st;
    const long long N = (long long)P.n_bytes;
    // longest segment a warp encodes: MEDIUM_MAX, or FEW_MEDIUM_MAX when the round has
    // no more records than CTAs (a warp walks a segment 32 positions at a time; with
    // CTAs to spare, a whole CTA takes each longer one)
    const long long mmax = d1 - d0 <= (unsigned long long)gridDim.x ? FEW_MEDIUM_MAX : MEDIUM_MAX;
    // ---- pass 1: warps
    for (;;) {
        unsigned long long r = 0;
        if (lane == 0) r = d0 + atomicAdd(&st->rec_ctr, 1ull);
        r = __shfl_sync(FULL_MASK, r, 0);
        if (r >= d1) break;
        const long long s0 = (long long)__ldcg(&P.recs[r].start);
        const long long d = P.n_docs > 1 ? warp_doc_from(P.doc_offs, (long long)__ldcg(&P.recs[r].doc), P.n_docs, s0) : 0;
        long long lim = next_struct_cut(P, d, s0);
        if (lim > N) lim = N;
        const long long scan_hi = min(lim, s0 + mmax + 1);
        const long long send = warp_first_nonjunction(P, C.jb, s0 + 1, scan_hi);
        if (send >= scan_hi && scan_hi < lim) {  // no cut within mmax + 1 bytes: a CTA or grid job
            if (lane == 0) {
                P.recs[r].count = REC_GIANT;
                P.glist[atomicAdd(&P.gscr[4], 1ull)] = (uint32_t)r;
            }
            continue;
        }
        encode_record(P, C, WarpGroup{}, r, s0, (unsigned long long)(send - s0), t0, par, lane == 0,
                      &C.w[wid].dl_arena, reinterpret_cast<uint32_t *>(&C.w[wid]), offsetof(WarpSmem, n_miss));
    }
    grid_sync(st, ++nbar);
    // ---- pass 2: several giants -> one CTA each (up to CTA_GIANT_MAX bytes), then
    //      every CTA together on each remaining giant, in record order
    //      (a lone one too when it is short: a pass of the grid engine costs three grid
    //      barriers, so 600 B of digits take 314 us on the grid and 130 us on one CTA
    //      in shared memory; the grid wins from ~6 KB)
    const unsigned long long n_giants = __ldcg(&P.gscr[4]);
    if (n_giants > 1 || (n_giants == 1 && GPUBPE_LONE_CTA_MAX > mmax)) {
        cta_giants(P, C, t0, par, n_giants > 1 ? CTA_GIANT_MAX : GPUBPE_LONE_CTA_MAX, mmax);
        grid_sync(st, ++nbar);
    }
    grid_giants(P, C, t0, par, nbar, mmax);
}

// ------------------------------------------------------------------ kernel

// Every exit of k_encode: the last CTA to leave copies the call's results
// (id count, overflow flag, counters) to P.mirror, pinned host memory mapped
// into the device, so a host call reads them after its synchronisation with
// no device-to-host copy (one DMA costs ~9 us of setup on this link).
//
// System-scope fences: every CTA's stores (ids and offsets in mapped host
// memory) reach the host before its exit count, and the mirror after all of
// them, so a host that sees the mirror may read the results without waiting
// for the stream to drain.
__device__ __forceinline__ void kernel_exit(const EncodeParams &P) {
    if (!P.mirror) return;
    __syncthreads();  // this CTA's stores and counter atomics are issued
    if (threadIdx.x == 0) {
        __threadfence_system();
        if (atomicAdd(&P.st->exit_ctr, 1ull) == gridDim.x - 1) {
            __threadfence_system();
            P.mirror->n_ids = __ldcg(&P.st->n_ids);
            P.mirror->overflow = __ldcg(&P.st->overflow);
            const unsigned long long *c = &P.st->c.n_segments;
            unsigned long long *d = &P.mirror->c.n_segments;
            for (int i = 0; i < (int)(sizeof(PassCounters) / 8); ++i) d[i] = __ldcg(&c[i]);
            __threadfence_system();
            *reinterpret_cast<volatile unsigned long long *>(&P.mirror->done) = P.mirror_tag;  // last
        }
    }
}

// kOneEach: the batch has at most one tile per warp (one round; tiles assigned
// statically).  A separate instantiation keeps the general kernel's code (and
// register allocation) exactly as tuned for many tiles per warp.
template <bool kOneEach>
__global__ void __launch_bounds__(NT, 1) k_encode(const __grid_constant__ EncodeParams P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    CtaSmem &C = *reinterpret_cast<CtaSmem *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    EncodeState *st = P.st;
    if (blockIdx.x == 0) {
        unsigned long long *z = reinterpret_cast<unsigned long long *>(P.st_next);
        for (int k = tid; k < (int)(sizeof(EncodeState) / 8); k += NT) z[k] = 0;
        if (tid == 0) P.gscr[4] = 0;  // giants of the round (appended after the round's first grid barrier)
    }
    if (kOneEach && !P.arrive) {  // this warp's tile bytes on their way to L2 while the bitmap loads
        const unsigned long long t = (unsigned long long)wid * gridDim.x + blockIdx.x;
        const int lane_ = tid & 31;
        if (t < P.n_tiles && lane_ * 128 < P.tile_bytes + HALO) {
            const unsigned long long at = t * (unsigned long long)P.tile_bytes + (unsigned long long)lane_ * 128;
            if (at < P.n_bytes) asm volatile("prefetch.global.L2 [%0];" ::"l"(P.bytes + at));
        }
    }
    for (int k = tid; k < 2048; k += NT) C.jb[k] = __ldg(&P.T.jbits[k]);
    for (int k = tid; k < 256; k += NT) C.base[k] = __ldg(&P.T.base[k]);
    if (tid < (int)(sizeof(PassCounters) / 8)) (&C.pc.n_segments)[tid] = 0;
    if (tid < 2) C.seen[tid] = 0;
    if (tid == 0) {
        C.arrived = 0;
        C.poll_lock = 0;
    }
    __syncthreads();
    if (P.dbg && tid == 0) P.dbg[4 * blockIdx.x] = gtimer();
    WarpSmem &S = C.w[wid];
    WarpCtx X{};
    unsigned int nbar = 0;
    unsigned long long d_done = 0, ng = 0;
    const unsigned long long R = P.round_tiles;
    const unsigned long long G = gridDim.x;
    for (unsigned long long r = 0, t0 = 0; t0 < P.n_tiles; ++r, t0 += R) {
        const unsigned long long t1 = min(P.n_tiles, t0 + R), par = r & 1;
        // ---- phase A: encode tiles of the round into their slots.  At most one
        //      tile per warp: tile = warp rank, interleaved across the SMs (no claim
        //      atomics); otherwise tiles are claimed from the round's counter.
        if constexpr (kOneEach) {
            // placement ranges of q tiles; a finished tile adds itself to its range's word
            const bool fast = G <= (unsigned long long)RNG_MAX;
            // (32-bit: one round holds at most G * NW tiles; a 64-bit division is ~60 instructions)
            const unsigned long long q = ((uint32_t)P.n_tiles + (uint32_t)G - 1) / (uint32_t)G;
            const unsigned long long t = t0 + (unsigned long long)wid * G + blockIdx.x;
            if (t < t1) {
                const unsigned long long g0 = P.dbg ? gtimer() : 0;
                const uint32_t tw = encode_tile(P, C, S, t, par * R + (t - t0), X);
                if (fast) {
                    __syncwarp();
                    // release (orders the warp's slot, tile word, document offsets and
                    // records before the add; no L1 invalidation, unlike __threadfence)
                    if (lane == 0) red_release_add(&st->rng[(uint32_t)t / (uint32_t)q], (1ull << 40) | TW_ENTRIES(tw));
                }
                if (P.dbg && lane == 0 && t < 4096) {
                    P.dbg[1024 + 2 * t] = g0;
                    P.dbg[1024 + 2 * t + 1] = gtimer();
                }
            }
            if (P.dbg_phase_a_only) return;
            if (fast) {
                warp_counters(C, X);  // final: summed by warp 1 after the completion barrier
                complete_one_round(P, C, q);
                if (P.dbg && tid == 0) P.dbg[4 * blockIdx.x + 2] = gtimer();
                if (C.bcast[3] == 0) {  // no deferred segments: place and finish
                    if (wid == 1) cta_counters(C, &st->c);
                    const unsigned long long lo = min(t1, blockIdx.x * q), hi = min(t1, lo + q);
                    if (P.dbg && tid == 0) P.dbg[36864 + 4 * blockIdx.x + 1] = gtimer();
                    if (hi > lo) place_range_one(P, C, lo, hi, C.bcast[0]);
                    if (P.dbg && tid == 0) P.dbg[4 * blockIdx.x + 3] = gtimer();
                    kernel_exit(P);
                    return;
                }
                // deferred segments: the general path below (every CTA read the same count)
            }
        } else {
            for (;;) {
                unsigned long long t = 0;
                if (lane == 0) t = t0 + atomicAdd(&st->actr[par], 1ull);
                t = __shfl_sync(FULL_MASK, t, 0);
                if (t >= t1) break;
                const unsigned long long g0 = P.dbg ? gtimer() : 0;
                encode_tile(P, C, S, t, par * R + (t - t0), X);
                if (P.dbg && lane == 0 && t < 4096) {
                    P.dbg[1024 + 2 * t] = g0;
                    P.dbg[1024 + 2 * t + 1] = gtimer();
                }
            }
        }
        if (P.dbg_phase_a_only) return;
        if (blockIdx.x == 0 && tid == 0) st->actr[par ^ 1] = 0;
        if (P.dbg && tid == 0 && r == 0) P.dbg[4 * blockIdx.x + 1] = gtimer();
        grid_sync(st, ++nbar, &C.bcast[3]);
        if (P.dbg && tid == 0 && r == 0) P.dbg[4 * blockIdx.x + 2] = gtimer();
        // ---- rare: deferred segments recorded in this round (count read with the barrier).
        //      When another round follows, a CTA that already left this barrier may append
        //      next-round records before a slower CTA polls, so the total comes from the
        //      per-parity counters instead (this round's parity is stable until the next
        //      barrier; the other one was read last round): every CTA sees the same D.
        unsigned long long D = C.bcast[3];
        if (!kOneEach && t1 < P.n_tiles) {  // (kOneEach: one round only)
            if (tid == 0) {
                C.seen[par] = ld_relaxed(&st->ndef[par]);
                C.bcast[3] = C.seen[0] + C.seen[1];
            }
            __syncthreads();
            D = C.bcast[3];
        }
        if (D > d_done) {
            if (D > P.rec_cap) {
                if (blockIdx.x == 0 && tid == 0) atomicExch(&st->overflow, 1ull);
                kernel_exit(P);
                return;
            }
            encode_deferred(P, C, d_done, D, t0, par, nbar);
            grid_sync(st, ++nbar);
            ng = __ldcg(&P.gscr[4]);
            if (blockIdx.x == 0 && tid == 0) {
                st->rec_ctr = 0;
                st->rec_ctr2 = 0;
            }
            if (__ldcg(&st->overflow)) {
                kernel_exit(P);
                return;
            }
            d_done = D;
        }
        // ---- phase B: place this CTA's contiguous range of the round's tiles
        const unsigned long long q = (t1 - t0 + G - 1) / G;
        const unsigned long long lo = min(t1, t0 + blockIdx.x * q), hi = min(t1, lo + q);
        // one round only: the counters are final here; publishing them before the
        // placement takes their atomics off the kernel's tail
        if constexpr (kOneEach) publish_counters(C, X, &st->c);
        if (P.dbg && tid == 0 && r == 0) P.dbg[36864 + 4 * blockIdx.x] = gtimer();
        place_range(P, C, r, t0, lo, hi);
        if (ng) {  // giants' ids: one grid-wide copy once their destinations are placed
            grid_sync(st, ++nbar);
            if (blockIdx.x == 0 && tid == 0) P.gscr[4] = 0;
            // (shorter results were copied by their tile's warp)
            if constexpr (kOneEach) {  // latency-sized calls: few giants, no extra code on the path
                for (unsigned long long gi = 0; gi < ng; ++gi) {
                    const DefRec *rec = &P.recs[__ldcg(&P.glist[gi])];
                    const uint32_t cnt = __ldcg(&rec->count);
                    if (cnt < GIANT_MIN - 1) continue;
                    const uint32_t *src = P.arena + __ldcg(&rec->res);
                    uint32_t *dst = P.out_ids + __ldcg(&rec->dst);
                    for (unsigned long long j = (unsigned long long)blockIdx.x * NT + tid; j < cnt;
                         j += (unsigned long long)gridDim.x * NT)
                        dst[j] = out_id(P.T, __ldcg(&src[j]));
                }
            } else
            for (unsigned long long gi0 = 0; gi0 < ng; gi0 += NT) {
                giant_masks(P, C, gi0, ng, [](const DefRec *rec) { return __ldcg(&rec->count) >= GIANT_MIN - 1; });
                for (int w = 0; w < NW; ++w)
                    for (uint32_t m = gmask(C)[w]; m; m &= m - 1) {
                        const DefRec *rec = &P.recs[__ldcg(&P.glist[gi0 + 32 * w + (__ffs(m) - 1)])];
                        const uint32_t cnt = __ldcg(&rec->count);
                        const uint32_t *src = P.arena + __ldcg(&rec->res);
                        uint32_t *dst = P.out_ids + __ldcg(&rec->dst);
                        for (unsigned long long j = (unsigned long long)blockIdx.x * NT + tid; j < cnt;
                             j += (unsigned long long)gridDim.x * NT)
                            dst[j] = out_id(P.T, __ldcg(&src[j]));
                    }
            }
            ng = 0;
        }
    }
    if constexpr (!kOneEach) publish_counters(C, X, &st->c);
    if (P.dbg && tid == 0) P.dbg[4 * blockIdx.x + 3] = gtimer();
    kernel_exit(P);
}

// ------------------------------------------------------------------ lookup

__global__ void k_lookup_pairs(DevTables T, const uint32_t *l, const uint32_t *r,
                               unsigned long long n, uint32_t *nw, uint32_t *rank) {
    unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    PairHit h = probe_pair(T, l[i], r[i]);
    rank[i] = h.rank;
    nw[i] = h.rank == GPUBPE_INF ? 0u : h.nw;
}

// ------------------------------------------------------------------ launchers

size_t tile_smem_bytes() { return sizeof(CtaSmem); }
int unit_max() { return UNIT_MAX; }

cudaError_t launch_encode(const EncodeParams &P, int grid, cudaStream_t s, cudaEvent_t *ev,
                          const cudaAccessPolicyWindow *win, bool coop) {
    if (ev) cudaEventRecord(ev[0], s);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = sizeof(CtaSmem);
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (coop) {
        attr[na].id = cudaLaunchAttributeCooperative;
        attr[na].val.cooperative = 1;
        ++na;
    }
    if (win && win->num_bytes) {
        attr[na].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[na].val.accessPolicyWindow = *win;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    const bool one_each = P.n_tiles <= (unsigned long long)grid * NW;  // one round, <= 1 tile per warp
    cudaError_t e = one_each ? cudaLaunchKernelEx(&cfg, k_encode<true>, P) : cudaLaunchKernelEx(&cfg, k_encode<false>, P);
    if (ev) cudaEventRecord(ev[1], s);
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t setup_kernels() {
    cudaError_t e = cudaFuncSetAttribute(k_encode<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sizeof(CtaSmem));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_encode<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)sizeof(CtaSmem));
}

cudaError_t tile_occupancy(int *blocks) {
    int b1 = 0, b2 = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b1, k_encode<true>, NT, sizeof(CtaSmem));
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b2, k_encode<false>, NT, sizeof(CtaSmem));
    *blocks = std::min(b1, b2);
    return e;
}

cudaError_t launch_lookup(const DevTables &T, const uint32_t *l, const uint32_t *r,
                          unsigned long long n, uint32_t *nw, uint32_t *rank, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_lookup_pairs<<<(unsigned int)((n + 255) / 256), 256, 0, s>>>(T, l, r, n, nw, rank);
    return cudaGetLastError();
}
