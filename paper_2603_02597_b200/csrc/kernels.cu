// kernels.cu -- encode kernels (see kernels.cuh for the pipeline).
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

#include "kernels.cuh"

// ------------------------------------------------------------------ helpers

// Last document d with offs[d] <= p (p < n_bytes): the non-empty doc holding p.
__device__ __forceinline__ long long doc_of(const long long *offs, unsigned long long n_docs,
                                            long long p) {
    long long lo = 0, hi = (long long)n_docs;
    while (lo < hi) {
        long long mid = (lo + hi + 1) >> 1;
        if (__ldg(&offs[mid]) <= p) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Smallest structural cut (doc end or chunk cut) strictly after p, where doc d
// holds p.
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

// Largest structural cut <= p (doc start or chunk cut), doc d holds p.
__device__ __forceinline__ long long prev_struct_cut(const EncodeParams &P, long long d, long long p) {
    long long s = __ldg(&P.doc_offs[d]), e = __ldg(&P.doc_offs[d + 1]);
    if ((unsigned long long)(e - s) > P.max_seq_len) {
        long long cb = (long long)P.chunk_budget;
        return s + ((p - s) / cb) * cb;
    }
    return s;
}

__device__ __forceinline__ bool junction_at(const EncodeParams &P, long long p) {
    return is_junction(P.T.jbits, __ldg(&P.bytes[p - 1]), __ldg(&P.bytes[p]));
}

// CTA: first p in [lo, hi) with a non-junction before p, else hi.
__device__ long long cta_first_nonjunction(const EncodeParams &P, long long lo, long long hi,
                                           EngineShared &sh) {
    for (long long b = lo; b < hi; b += NT) {
        long long p = b + threadIdx.x;
        bool f = p < hi && !junction_at(P, p);
        unsigned long long k = f ? (unsigned long long)p : ~0ull;
        unsigned long long m = block_min_u64(k, sh);
        if (m != ~0ull) return (long long)m;
    }
    return hi;
}

// CTA: last p in (lo, hi] with a non-junction before p, else lo.
__device__ long long cta_last_nonjunction(const EncodeParams &P, long long lo, long long hi,
                                          EngineShared &sh) {
    for (long long b = hi; b > lo; b -= NT) {
        long long p = b - threadIdx.x;
        bool f = p > lo && !junction_at(P, p);
        unsigned long long k = f ? ~(unsigned long long)p : ~0ull;  // min of ~p = max p
        unsigned long long m = block_min_u64(k, sh);
        if (m != ~0ull) return (long long)(~m);
    }
    return lo;
}

// ------------------------------------------------------------------ K0

__global__ void __launch_bounds__(NT) k_windows(EncodeParams P) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        EncodeState *s = P.st;
        s->tile_counter = 0; s->n_giant = 0; s->arena_used = 0; s->overflow = 0; s->error = 0;
        s->n_ids = 0; s->n_segments = 0; s->memo_hits = 0; s->short_merges = 0;
        s->medium_segments = 0; s->giant_segments = 0; s->giant_bytes = 0; s->engine_passes = 0;
    }
    unsigned long long w = (unsigned long long)blockIdx.x * NT + threadIdx.x;
    if (w >= P.n_win) return;
    const long long N = (long long)P.n_bytes;
    long long a = (long long)(w * WIN);
    long long d = doc_of(P.doc_offs, P.n_docs, a);
    P.window_doc[w] = d;
    P.giant_at[w] = -1;
    // slots (a, a+WIN]: is any of them a boundary?
    long long hi = a + WIN;
    bool clear = hi < N && next_struct_cut(P, d, a) > hi;
    if (clear) {
        uint32_t x = __ldg(&P.bytes[a]);
        for (long long p = a + 1; p <= hi; ++p) {
            uint32_t y = __ldg(&P.bytes[p]);
            if (!is_junction(P.T.jbits, x, y)) { clear = false; break; }
            x = y;
        }
    }
    P.wclear[w] = clear;
}

// ------------------------------------------------------------------ K1

__global__ void __launch_bounds__(NT) k_giant(EncodeParams P) {
    __shared__ EngineShared sh;
    __shared__ unsigned int found[NT];
    __shared__ unsigned int n_found;
    const long long N = (long long)P.n_bytes;
    for (unsigned long long w0 = (unsigned long long)blockIdx.x * NT; w0 < P.n_win;
         w0 += (unsigned long long)gridDim.x * NT) {
        if (threadIdx.x == 0) n_found = 0;
        __syncthreads();
        unsigned long long w = w0 + threadIdx.x;
        if (w < P.n_win && P.wclear[w] && (w == 0 || !P.wclear[w - 1]))
            found[atomicAdd(&n_found, 1u)] = threadIdx.x;
        __syncthreads();
        const unsigned int nf = n_found;
        for (unsigned int f = 0; f < nf; ++f) {
            const unsigned long long wr = w0 + found[f];
            const long long a = (long long)(wr * WIN);
            // exact start: largest boundary <= a
            long long d = P.window_doc[wr];
            long long lo = prev_struct_cut(P, d, a);
            long long s = cta_last_nonjunction(P, lo, a, sh);
            // run of clear windows [wr, w2]
            unsigned long long w2 = wr;
            for (;;) {
                unsigned long long q = w2 + 1 + threadIdx.x;
                bool stop = q >= P.n_win || !P.wclear[q];
                unsigned long long k = stop ? q : ~0ull;
                unsigned long long m = block_min_u64(k, sh);
                if (m != ~0ull) { w2 = m - 1; break; }
                w2 += NT;
            }
            // exact end: smallest boundary > q0 = (w2+1)*WIN  (q0 < N)
            long long q0 = (long long)((w2 + 1) * WIN);
            long long d2 = doc_of(P.doc_offs, P.n_docs, q0);
            long long lim = next_struct_cut(P, d2, q0);
            if (lim > N) lim = N;
            long long e = cta_first_nonjunction(P, q0 + 1, lim, sh);
            const unsigned long long L = (unsigned long long)(e - s);
            // arena: tok, tok2 (u32), pr, pr2 (uint2), sel (u8)
            const unsigned long long words = (L * 25 + 15) / 16 * 4;  // u32 units, 16 B aligned
            __shared__ unsigned long long sh_off, sh_rec;
            if (threadIdx.x == 0) {
                unsigned long long off = atomicAdd(&P.st->arena_used, words);
                if ((off + words) * 4 > P.arena_cap) {
                    atomicExch(&P.st->overflow, 1ull);
                    off = ~0ull;
                }
                sh_off = off;
                unsigned long long rec = atomicAdd(&P.st->n_giant, 1ull);
                sh_rec = rec;
                P.recs[rec].start = (unsigned long long)s;
                P.recs[rec].end = (unsigned long long)e;
                P.recs[rec].count = 0;
                P.recs[rec].out_off = 0;
                P.giant_at[s / WIN] = (int)rec;
                atomicAdd(&P.st->giant_segments, 1ull);
                atomicAdd(&P.st->giant_bytes, L);
            }
            __syncthreads();
            const unsigned long long off = sh_off, rec = sh_rec;
            if (off != ~0ull) {
                uint32_t *base = reinterpret_cast<uint32_t *>(P.arena) + off;
                EngineMem M;
                M.tok = base;
                M.tok2 = base + L;
                M.pr = reinterpret_cast<uint2 *>(base + 2 * L + (2 * L & 1));
                M.pr2 = M.pr + L;
                M.sel = reinterpret_cast<uint8_t *>(M.pr2 + L);
                for (unsigned long long j = threadIdx.x; j < L; j += NT)
                    M.tok[j] = __ldg(&P.T.base[__ldg(&P.bytes[s + j])]);
                __syncthreads();
                uint32_t passes;
                const uint32_t *res;
                uint32_t cnt = engine_run(P.T, M, (uint32_t)L, P.strict || !P.T.well_formed, sh,
                                          &passes, &res);
                if (threadIdx.x == 0) {
                    P.recs[rec].count = cnt;
                    P.recs[rec].out_off = (unsigned long long)(res - reinterpret_cast<uint32_t *>(P.arena));
                    atomicAdd(&P.st->engine_passes, (unsigned long long)passes);
                }
            }
            __syncthreads();
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ K2

struct TileSmem {
    uint8_t sb[LD + 16];
    uint32_t bits[(LD + 31) / 32 + 2];
    uint32_t sid[LD];
    uint32_t srk[LD];
    uint32_t snw[LD];
    uint16_t seg_start[TILE];
    uint16_t seg_end[TILE];
    uint32_t seg_cnt[TILE];
    uint16_t pend[TILE / (SHORT_MAX + 1) + 4];
    EngineShared es;
    unsigned long long tile;
    unsigned long long base;  // exclusive output prefix of this tile
    unsigned int n_seg, n_pend, total;
    int ovh_kind;            // 0 none, 1 medium (result in med buffer), 2 giant
    unsigned int ovh_seg;    // segment index of the overhang segment
    unsigned long long ovh_src;  // giant: arena element offset; medium: pointer offset
    unsigned int c_memo, c_short, c_med;
};

// Per-thread exact greedy (reference order) on sid[k0..k0+len) -- any table.
__device__ uint32_t thread_greedy(const DevTables &T, uint32_t *tok, uint32_t *rk, uint32_t *nw,
                                  uint32_t n) {
    for (uint32_t j = 0; j + 1 < n; ++j) {
        PairHit h = probe_pair(T, tok[j], tok[j + 1]);
        rk[j] = h.rank;
        nw[j] = h.nw;
    }
    for (;;) {
        uint32_t best = GPUBPE_INF, p = 0;
        for (uint32_t j = 0; j + 1 < n; ++j)
            if (rk[j] < best) { best = rk[j]; p = j; }
        if (best == GPUBPE_INF) break;
        tok[p] = nw[p];
        for (uint32_t j = p + 1; j + 1 < n; ++j) tok[j] = tok[j + 1];
        for (uint32_t j = p + 1; j + 2 < n; ++j) { rk[j] = rk[j + 1]; nw[j] = nw[j + 1]; }
        --n;
        if (p > 0) {
            PairHit h = probe_pair(T, tok[p - 1], tok[p]);
            rk[p - 1] = h.rank; nw[p - 1] = h.nw;
        }
        if (p + 1 < n) {
            PairHit h = probe_pair(T, tok[p], tok[p + 1]);
            rk[p] = h.rank; nw[p] = h.nw;
        }
    }
    return n;
}

// Memo probe for sb[0..len), 2 <= len <= SHORT_MAX.  Returns id or INF.
__device__ uint32_t memo_lookup(const DevTables &T, const uint8_t *sb, uint32_t len) {
    unsigned long long lo = 0;
    uint32_t m = len < 8 ? len : 8;
    for (uint32_t j = 0; j < m; ++j) lo |= (unsigned long long)sb[j] << (8 * j);
    unsigned long long h = memo_hash_step(memo_hash_init(len), lo);
    for (uint32_t c = 8; c < len; c += 8) {
        unsigned long long ch = 0;
        for (uint32_t j = c; j < len && j < c + 8; ++j) ch |= (unsigned long long)sb[j] << (8 * (j - c));
        h = memo_hash_step(h, ch);
    }
    uint32_t slot = (uint32_t)h & T.memo_mask;
    for (;;) {
        uint4 e = __ldg(&T.memo[slot]);
        if (e.w == 0) return GPUBPE_INF;
        if ((e.w & 0xFFu) == len && e.x == (uint32_t)lo && e.y == (uint32_t)(lo >> 32)) {
            bool eq = true;
            if (len > 8) {
                const uint8_t *tail = T.blob + (e.w >> 8);
                for (uint32_t j = 8; j < len; ++j)
                    if (__ldg(&tail[j]) != sb[j]) { eq = false; break; }
            }
            if (eq) return e.z;
        }
        slot = (slot + 1) & T.memo_mask;
    }
}

__device__ __forceinline__ void publish(unsigned long long *w, unsigned long long v) {
    cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> r(*w);
    r.store(v, cuda::memory_order_release);
}
__device__ __forceinline__ unsigned long long peek(unsigned long long *w) {
    cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> r(*w);
    return r.load(cuda::memory_order_acquire);
}

#define LB_AGG 1ull
#define LB_INC 2ull
#define LB_VALUE_MASK ((1ull << 42) - 1)

__global__ void __launch_bounds__(NT) k_tile(EncodeParams P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TileSmem &S = *reinterpret_cast<TileSmem *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const long long N = (long long)P.n_bytes;
    const DevTables &T = P.T;
    const bool strict = P.strict || !T.well_formed;
    const bool use_memo = T.memo_mask != 0;
    uint8_t *medp = P.med_scratch + (size_t)blockIdx.x * MED_BYTES;
    EngineMem MM;
    MM.tok = reinterpret_cast<uint32_t *>(medp);
    MM.tok2 = MM.tok + MED_MAX;
    MM.pr = reinterpret_cast<uint2 *>(MM.tok2 + MED_MAX);
    MM.pr2 = MM.pr + MED_MAX;
    MM.sel = reinterpret_cast<uint8_t *>(MM.pr2 + MED_MAX);

    for (;;) {
        if (tid == 0) {
            S.tile = atomicAdd(&P.st->tile_counter, 1ull);
            S.n_pend = 0;
            S.ovh_kind = 0;
            S.c_memo = S.c_short = S.c_med = 0;
        }
        __syncthreads();
        const unsigned long long t = S.tile;
        if (t >= P.n_tiles) break;
        const long long a = (long long)(t * TILE);
        const long long b = min(a + TILE, N);
        const long long el = min(b + HALO, N);
        const int nld = (int)(el - a);
        const int ntile = (int)(b - a);

        // ---- load bytes
        for (int k = tid; k < nld; k += NT) S.sb[k] = __ldg(&P.bytes[a + k]);
        const uint32_t prev = a > 0 ? __ldg(&P.bytes[a - 1]) : 0u;
        __syncthreads();
        // ---- junction bits for slots [0, nld); slot k is the cut before a+k
        for (int w = wid; w * 32 < nld + 1; w += NT / 32) {
            int k = w * 32 + lane;
            bool cut;
            if (k < nld) {
                uint32_t x = k ? S.sb[k - 1] : prev;
                cut = (a + k == 0) || !is_junction(T.jbits, x, S.sb[k]);
            } else {
                cut = (k == nld) && (el == N);
            }
            unsigned m = __ballot_sync(0xffffffffu, cut);
            if (lane == 0) S.bits[w] = m;
        }
        __syncthreads();
        // ---- document starts and chunk cuts inside [a, el)
        {
            const long long d0 = P.window_doc[a / WIN];
            for (long long d = d0 + tid; d < (long long)P.n_docs; d += NT) {
                long long s = __ldg(&P.doc_offs[d]);
                if (s >= el) break;
                long long e = __ldg(&P.doc_offs[d + 1]);
                if (s >= a) { int k = (int)(s - a); atomicOr(&S.bits[k >> 5], 1u << (k & 31)); }
                if ((unsigned long long)(e - s) > P.max_seq_len) {
                    long long cb = (long long)P.chunk_budget;
                    long long m = s < a ? (a - s + cb - 1) / cb : 1;
                    if (m < 1) m = 1;
                    for (long long c = s + m * cb; c < e && c < el; c += cb) {
                        int k = (int)(c - a);
                        atomicOr(&S.bits[k >> 5], 1u << (k & 31));
                    }
                }
            }
        }
        __syncthreads();
        // ---- segments starting in [0, ntile)
        {
            const int per = TILE / NT;  // 8 slots per thread
            const int k0 = tid * per;
            uint32_t word = S.bits[k0 >> 5] >> (k0 & 31);
            uint32_t mine = word & ((1u << per) - 1);
            if (k0 >= ntile) mine = 0;
            else if (k0 + per > ntile) mine &= (1u << (ntile - k0)) - 1;
            uint32_t tot;
            uint32_t idx = block_excl_sum(__popc(mine), S.es, &tot);
            while (mine) {
                int bit = __ffs(mine) - 1;
                mine &= mine - 1;
                int k = k0 + bit;
                // next boundary after k
                int q = k + 1;
                int end = NOSEG;
                int lim = el == N ? nld : nld - 1;  // slots known: [0, nld) (+ nld at end of data)
                while (q <= lim) {
                    uint32_t wv = S.bits[q >> 5] >> (q & 31);
                    if (wv) {
                        int c = q + __ffs(wv) - 1;
                        if (c <= lim) end = c;
                        break;
                    }
                    q = (q | 31) + 1;
                }
                S.seg_start[idx] = (uint16_t)k;
                S.seg_end[idx] = (uint16_t)end;
                ++idx;
            }
            if (tid == 0) S.n_seg = tot;
        }
        __syncthreads();
        const unsigned int n_seg = S.n_seg;
        // ---- short segments: one thread each
        for (unsigned int i = tid; i < n_seg; i += NT) {
            const uint32_t k0 = S.seg_start[i], e = S.seg_end[i];
            if (e == NOSEG || e - k0 > SHORT_MAX) {
                S.seg_cnt[i] = PENDING;
                S.pend[atomicAdd(&S.n_pend, 1u)] = (uint16_t)i;
                continue;
            }
            const uint32_t len = e - k0;
            uint32_t cnt;
            if (len == 1) {
                S.sid[k0] = __ldg(&T.base[S.sb[k0]]);
                cnt = 1;
            } else {
                uint32_t id = use_memo ? memo_lookup(T, S.sb + k0, len) : GPUBPE_INF;
                if (id != GPUBPE_INF) {
                    S.sid[k0] = id;
                    cnt = 1;
                    atomicAdd(&S.c_memo, 1u);
                } else {
                    for (uint32_t j = 0; j < len; ++j) S.sid[k0 + j] = __ldg(&T.base[S.sb[k0 + j]]);
                    cnt = thread_greedy(T, S.sid + k0, S.srk + k0, S.snw + k0, len);
                    atomicAdd(&S.c_short, 1u);
                }
            }
            S.seg_cnt[i] = cnt;
        }
        __syncthreads();
        // ---- medium / overhang / giant segments: whole CTA, one at a time.
        // In-tile ones first (results land in sid); the overhang segment (end
        // past the loaded bytes, at most one per tile) last, its result stays
        // in the medium scratch (or the giant arena) until the store.
        const unsigned int n_pend = S.n_pend;
        for (int phase = 0; phase < 2; ++phase) {
            for (unsigned int pi = 0; pi < n_pend; ++pi) {
                const unsigned int i = S.pend[pi];
                const uint32_t k0 = S.seg_start[i], e = S.seg_end[i];
                if ((e == NOSEG) != (phase == 1)) continue;
                const long long s = a + k0;
                int rec = -1;
                if (e == NOSEG || e - k0 > WIN) {
                    int r = P.giant_at[s / WIN];
                    if (r >= 0 && (long long)P.recs[r].start == s) rec = r;
                }
                if (rec >= 0) {
                    const uint32_t cnt = (uint32_t)P.recs[rec].count;
                    const uint32_t *src = reinterpret_cast<const uint32_t *>(P.arena) + P.recs[rec].out_off;
                    if (e != NOSEG) {
                        for (uint32_t j = tid; j < cnt; j += NT) S.sid[k0 + j] = src[j];
                    } else if (tid == 0) {
                        S.ovh_kind = 2;
                        S.ovh_seg = i;
                        S.ovh_src = P.recs[rec].out_off;
                    }
                    if (tid == 0) S.seg_cnt[i] = cnt;
                    __syncthreads();
                    continue;
                }
                long long send;
                if (e != NOSEG) {
                    send = s + (e - k0);
                } else {
                    // overhang: scan for the end past the loaded bytes
                    long long d = doc_of(P.doc_offs, P.n_docs, s);
                    long long lim = next_struct_cut(P, d, s);
                    if (lim > N) lim = N;
                    send = cta_first_nonjunction(P, a + nld, lim, S.es);
                }
                const uint32_t len = (uint32_t)(send - s);
                if (len >= MED_MAX) {  // impossible for a non-giant segment
                    if (tid == 0) { atomicExch(&P.st->error, 1ull); S.seg_cnt[i] = 0; }
                    __syncthreads();
                    continue;
                }
                for (uint32_t j = tid; j < len; j += NT)
                    MM.tok[j] = __ldg(&T.base[e != NOSEG ? S.sb[k0 + j] : __ldg(&P.bytes[s + j])]);
                __syncthreads();
                uint32_t passes;
                const uint32_t *res;
                uint32_t cnt = engine_run(T, MM, len, strict, S.es, &passes, &res);
                if (e != NOSEG)
                    for (uint32_t j = tid; j < cnt; j += NT) S.sid[k0 + j] = res[j];
                if (tid == 0) {
                    S.seg_cnt[i] = cnt;
                    S.c_med++;
                    atomicAdd(&P.st->engine_passes, (unsigned long long)passes);
                    if (e == NOSEG) {
                        S.ovh_kind = 1;
                        S.ovh_seg = i;
                        S.ovh_src = (unsigned long long)(res - MM.tok);
                    }
                }
                __syncthreads();
            }
        }
        // ---- exclusive scan of counts -> seg_cnt becomes offsets
        {
            const int per = TILE / NT;
            uint32_t v[TILE / NT];
            uint32_t sum = 0;
#pragma unroll
            for (int j = 0; j < per; ++j) {
                unsigned int i = tid * per + j;
                v[j] = i < n_seg ? S.seg_cnt[i] : 0u;
                sum += v[j];
            }
            uint32_t tot;
            uint32_t off = block_excl_sum(sum, S.es, &tot);
#pragma unroll
            for (int j = 0; j < per; ++j) {
                unsigned int i = tid * per + j;
                if (i < n_seg) S.seg_cnt[i] = off;
                off += v[j];
            }
            if (tid == 0) S.total = tot;
        }
        __syncthreads();
        // ---- decoupled look-back
        const unsigned long long total = S.total;
        const unsigned long long tag = (unsigned long long)P.epoch << 44;
        if (wid == 0) {
            unsigned long long excl = 0;
            if (t == 0) {
                if (lane == 0) publish(&P.status[0], tag | (LB_INC << 42) | total);
            } else {
                if (lane == 0) publish(&P.status[t], tag | (LB_AGG << 42) | total);
                long long pos = (long long)t - 1;
                for (;;) {
                    long long j = pos - lane;
                    unsigned long long v;
                    unsigned long long flag;
                    if (j >= 0) {
                        do {
                            v = peek(&P.status[j]);
                            flag = ((v >> 44) == P.epoch) ? ((v >> 42) & 3ull) : 0ull;
                        } while (flag == 0);
                    } else {
                        v = LB_INC << 42;
                        flag = LB_INC;
                    }
                    unsigned inc = __ballot_sync(0xffffffffu, flag == LB_INC);
                    int stop = inc ? __ffs(inc) - 1 : 31;
                    unsigned long long val = (lane <= stop) ? (v & LB_VALUE_MASK) : 0ull;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
                    excl += val;
                    if (inc) break;
                    pos -= 32;
                }
                if (lane == 0) publish(&P.status[t], tag | (LB_INC << 42) | (excl + total));
            }
            if (lane == 0) S.base = excl;
        }
        __syncthreads();
        const unsigned long long base = S.base;
        // ---- store ids
        uint32_t *out = P.out_ids + base;
        const int okind = S.ovh_kind;
        const unsigned int oseg = S.ovh_seg;
        for (unsigned int i = tid; i < n_seg; i += NT) {
            if (okind && i == oseg) continue;
            const uint32_t k0 = S.seg_start[i];
            const uint32_t o = S.seg_cnt[i];
            const uint32_t c = (i + 1 < n_seg ? S.seg_cnt[i + 1] : S.total) - o;
            for (uint32_t j = 0; j < c; ++j) out[o + j] = out_id(T, S.sid[k0 + j]);
        }
        if (okind) {
            const uint32_t o = S.seg_cnt[oseg];
            const uint32_t c = (oseg + 1 < n_seg ? S.seg_cnt[oseg + 1] : S.total) - o;
            const uint32_t *src = okind == 2
                ? reinterpret_cast<const uint32_t *>(P.arena) + S.ovh_src
                : MM.tok + S.ovh_src;
            for (uint32_t j = tid; j < c; j += NT) out[o + j] = out_id(T, src[j]);
        }
        // ---- document offsets for docs starting in [a, b) (or at N for the last tile)
        {
            const long long d0 = P.window_doc[a / WIN];
            const long long hi = (b == N) ? N + 1 : b;
            for (long long d = d0 + tid; d <= (long long)P.n_docs; d += NT) {
                long long s = __ldg(&P.doc_offs[d]);
                if (s >= hi) break;
                if (s < a) continue;
                unsigned long long v;
                if (s == N) {
                    v = base + total;
                } else {
                    // segment starting at s - a
                    int k = (int)(s - a);
                    unsigned int lo = 0, hi2 = n_seg;
                    while (lo < hi2) {
                        unsigned int mid = (lo + hi2) >> 1;
                        if (S.seg_start[mid] < k) lo = mid + 1; else hi2 = mid;
                    }
                    v = base + (lo < n_seg ? S.seg_cnt[lo] : S.total);
                }
                P.out_offs[d] = (long long)v;
            }
        }
        if (tid == 0) {
            atomicAdd(&P.st->n_segments, (unsigned long long)n_seg);
            if (S.c_memo) atomicAdd(&P.st->memo_hits, (unsigned long long)S.c_memo);
            if (S.c_short) atomicAdd(&P.st->short_merges, (unsigned long long)S.c_short);
            if (S.c_med) atomicAdd(&P.st->medium_segments, (unsigned long long)S.c_med);
            if (b == N) atomicAdd(&P.st->n_ids, base + total);
        }
        __syncthreads();
    }
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

size_t tile_smem_bytes() { return sizeof(TileSmem); }

cudaError_t launch_encode(const EncodeParams &P, int grid_tile, int grid_giant, cudaStream_t s) {
    unsigned int gw = (unsigned int)((P.n_win + NT - 1) / NT);
    k_windows<<<gw, NT, 0, s>>>(P);
    k_giant<<<grid_giant, NT, 0, s>>>(P);
    k_tile<<<grid_tile, NT, sizeof(TileSmem), s>>>(P);
    return cudaGetLastError();
}

cudaError_t setup_kernels() {
    return cudaFuncSetAttribute(k_tile, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)sizeof(TileSmem));
}

cudaError_t tile_occupancy(int *blocks) {
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, k_tile, NT, sizeof(TileSmem));
}

cudaError_t launch_lookup(const DevTables &T, const uint32_t *l, const uint32_t *r,
                          unsigned long long n, uint32_t *nw, uint32_t *rank, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_lookup_pairs<<<(unsigned int)((n + 255) / 256), 256, 0, s>>>(T, l, r, n, nw, rank);
    return cudaGetLastError();
}
