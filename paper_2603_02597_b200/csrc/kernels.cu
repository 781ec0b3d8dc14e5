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

// ------------------------------------------------------------------ helpers

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
// document holding byte p.  32-ary search, all lanes get the result.
__device__ long long warp_doc_of(const long long *offs, unsigned long long n_docs, long long p) {
    const int lane = threadIdx.x & 31;
    long long lo = 0, hi = (long long)n_docs - 1;  // answer in [lo, hi]
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

// CTA: first p in [lo, hi) whose cut slot is a junction miss, else hi.
// Each thread checks 16 consecutive slots per round (4096 per round).
__device__ long long cta_first_nonjunction(const EncodeParams &P, long long lo, long long hi,
                                           EngineShared &sh) {
    for (long long b = lo; b < hi; b += 16 * NT) {
        const long long p0 = b + 16 * (long long)threadIdx.x;
        unsigned long long k = ~0ull;
        if (p0 < hi) {
            uint32_t x = __ldg(&P.bytes[p0 - 1]);
            const long long pe = min(p0 + 16, hi);
            for (long long p = p0; p < pe; ++p) {
                const uint32_t y = __ldg(&P.bytes[p]);
                if (!is_junction(P.T.jbits, x, y)) { k = (unsigned long long)p; break; }
                x = y;
            }
        }
        const unsigned long long m = block_min_u64(k, sh);
        if (m != ~0ull) return (long long)m;
    }
    return hi;
}

__device__ __forceinline__ void st_relaxed(unsigned long long *w, unsigned long long v) {
    cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> r(*w);
    r.store(v, cuda::memory_order_relaxed);
}
__device__ __forceinline__ unsigned long long ld_relaxed(unsigned long long *w) {
    cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> r(*w);
    return r.load(cuda::memory_order_relaxed);
}

// Memo probe for sb[0..len), 2 <= len <= SHORT_MAX.  Returns the id or INF.
__device__ uint32_t memo_lookup(const DevTables &T, const uint8_t *sb, uint32_t len) {
    unsigned long long lo = 0;
    const uint32_t m = len < 8 ? len : 8;
    for (uint32_t j = 0; j < m; ++j) lo |= (unsigned long long)sb[j] << (8 * j);
    unsigned long long h = memo_hash_step(memo_hash_init(len), lo);
    for (uint32_t c = 8; c < len; c += 8) {
        unsigned long long ch = 0;
        for (uint32_t j = c; j < len && j < c + 8; ++j) ch |= (unsigned long long)sb[j] << (8 * (j - c));
        h = memo_hash_step(h, ch);
    }
    uint32_t slot = (uint32_t)h & T.memo_mask;
    for (;;) {
        const uint4 e = __ldg(&T.memo[slot]);
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

// ------------------------------------------------------------------ kernel

struct TileSmem {
    uint8_t sb[LD + 16];
    uint32_t bits[(LD + 31) / 32 + 2];
    uint32_t sid[LD];  // ids of each segment, stored from the segment's start slot
    uint16_t seg_start[TILE];
    uint16_t seg_end[TILE];
    uint32_t seg_cnt[TILE];  // counts, then exclusive offsets
    uint16_t miss[TILE];     // segments for the warp engine
    uint16_t pend[TILE / (SHORT_MAX + 1) + 4];
    EngineShared es;
    unsigned long long tile;
    unsigned long long base;
    unsigned long long arena_off;
    long long d0;
    const uint32_t *ovh_src;  // result of the overhang segment (scratch or arena)
    unsigned int n_seg, n_miss, n_pend, total, ovh_seg;
    unsigned int c_memo, c_warp, c_med, c_giant, c_passes;
    unsigned long long c_giant_bytes;
};

__device__ __forceinline__ void set_bit(uint32_t *bits, int k) { atomicOr(&bits[k >> 5], 1u << (k & 31)); }

#define LB_AGG 1ull
#define LB_INC 2ull
#define LB_VALUE_MASK ((1ull << 42) - 1)

__global__ void __launch_bounds__(NT) k_encode(EncodeParams P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TileSmem &S = *reinterpret_cast<TileSmem *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const long long N = (long long)P.n_bytes;
    const DevTables &T = P.T;
    const bool strict = P.strict || !T.well_formed;
    const bool use_memo = T.memo_mask != 0;
    uint8_t *medp = P.med_scratch + (size_t)blockIdx.x * MED_BYTES;
    if (blockIdx.x == 0 && tid == 0) *P.st_next = EncodeState{};

    for (;;) {
        if (tid == 0) {
            S.tile = atomicAdd(&P.st->tile_counter, 1ull);
            S.n_miss = S.n_pend = 0;
            S.ovh_src = nullptr;
            S.ovh_seg = 0xFFFFFFFFu;
            S.c_memo = S.c_warp = S.c_med = S.c_giant = S.c_passes = 0;
            S.c_giant_bytes = 0;
        }
        __syncthreads();
        const unsigned long long t = S.tile;
        if (t >= P.n_tiles) break;
        const long long a = (long long)(t * TILE);
        const long long b = min(a + TILE, N);
        const long long el = min(b + HALO, N);
        const int nld = (int)(el - a);
        const int ntile = (int)(b - a);

        // ---- stage bytes; warp 0 finds the document holding byte a
        for (int k = tid; k < nld; k += NT) S.sb[k] = __ldg(&P.bytes[a + k]);
        const uint32_t prev = a > 0 ? __ldg(&P.bytes[a - 1]) : 0u;
        if (wid == 0) {
            const long long d = P.n_docs > 1 ? warp_doc_of(P.doc_offs, P.n_docs, a) : 0;
            if (lane == 0) S.d0 = d;
        }
        __syncthreads();
        // ---- junction-miss bits for slots [0, nld); slot k = cut before byte a+k
        for (int w = wid; w * 32 < nld + 1; w += NT / 32) {
            const int k = w * 32 + lane;
            bool cut;
            if (k < nld) {
                const uint32_t x = k ? S.sb[k - 1] : prev;
                cut = (a + k == 0) || !is_junction(T.jbits, x, S.sb[k]);
            } else {
                cut = (k == nld) && (el == N);
            }
            const unsigned m = __ballot_sync(FULL_MASK, cut);
            if (lane == 0) S.bits[w] = m;
        }
        __syncthreads();
        // ---- document starts and chunk cuts inside [a, el)
        const long long d0 = S.d0;
        for (long long d = d0 + tid; d < (long long)P.n_docs; d += NT) {
            const long long s = __ldg(&P.doc_offs[d]);
            if (s >= el) break;
            const long long e = __ldg(&P.doc_offs[d + 1]);
            if (s >= a) set_bit(S.bits, (int)(s - a));
            if ((unsigned long long)(e - s) > P.max_seq_len) {
                const long long cb = (long long)P.chunk_budget;
                long long m = s < a ? (a - s + cb - 1) / cb : 1;
                if (m < 1) m = 1;
                for (long long c = s + m * cb; c < e && c < el; c += cb) set_bit(S.bits, (int)(c - a));
            }
        }
        __syncthreads();
        // ---- segments starting in [0, ntile): start and end slot
        {
            const int per = TILE / NT;
            const int k0 = tid * per;
            uint32_t mine = (S.bits[k0 >> 5] >> (k0 & 31)) & ((1u << per) - 1);
            if (k0 >= ntile) mine = 0;
            else if (k0 + per > ntile) mine &= (1u << (ntile - k0)) - 1;
            uint32_t tot;
            uint32_t idx = block_excl_sum(__popc(mine), S.es, &tot);
            const int lim = el == N ? nld : nld - 1;  // last slot whose cut status is known
            while (mine) {
                const int k = k0 + __ffs(mine) - 1;
                mine &= mine - 1;
                int q = k + 1, end = NOSEG;
                while (q <= lim) {
                    const uint32_t wv = S.bits[q >> 5] >> (q & 31);
                    if (wv) {
                        const int c = q + __ffs(wv) - 1;
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
        // ---- one thread per segment: base id, memo, or defer
        for (unsigned int i = tid; i < n_seg; i += NT) {
            const uint32_t k0 = S.seg_start[i], e = S.seg_end[i];
            if (e == NOSEG || e - k0 > SHORT_MAX) {
                S.pend[atomicAdd(&S.n_pend, 1u)] = (uint16_t)i;
                continue;
            }
            const uint32_t len = e - k0;
            if (len == 1) {
                S.sid[k0] = __ldg(&T.base[S.sb[k0]]);
                S.seg_cnt[i] = 1;
                continue;
            }
            const uint32_t id = use_memo ? memo_lookup(T, S.sb + k0, len) : GPUBPE_INF;
            if (id != GPUBPE_INF) {
                S.sid[k0] = id;
                S.seg_cnt[i] = 1;
                atomicAdd(&S.c_memo, 1u);
            } else {
                S.miss[atomicAdd(&S.n_miss, 1u)] = (uint16_t)i;
            }
        }
        __syncthreads();
        // ---- one warp per memo miss: exact multi-merge in registers
        {
            const unsigned int n_miss = S.n_miss;
            unsigned int wp = 0, ws = 0;
            for (unsigned int m = wid; m < n_miss; m += NT / 32) {
                const unsigned int i = S.miss[m];
                const uint32_t k0 = S.seg_start[i], len = S.seg_end[i] - k0;
                const uint32_t tk = lane < len ? __ldg(&T.base[S.sb[k0 + lane]]) : 0u;
                uint32_t np;
                const uint32_t cnt = warp_bpe(T, tk, len, strict, S.sid + k0, &np);
                wp += np;
                ++ws;
                if (lane == 0) S.seg_cnt[i] = cnt;
            }
            if (lane == 0 && ws) {
                atomicAdd(&S.c_passes, wp);
                atomicAdd(&S.c_warp, ws);
            }
        }
        __syncthreads();
        // ---- long segments: whole CTA, in-tile ones first, the overhang last
        const unsigned int n_pend = S.n_pend;
        for (int phase = 0; phase < 2; ++phase) {
            for (unsigned int pi = 0; pi < n_pend; ++pi) {
                const unsigned int i = S.pend[pi];
                const uint32_t k0 = S.seg_start[i], e = S.seg_end[i];
                if ((e == NOSEG) != (phase == 1)) continue;
                const long long s = a + k0;
                long long send;
                if (e != NOSEG) {
                    send = s + (e - k0);
                } else {
                    long long d = d0;
                    while (__ldg(&P.doc_offs[d + 1]) <= s) ++d;  // docs overlapping the tile
                    long long lim = next_struct_cut(P, d, s);
                    if (lim > N) lim = N;
                    send = cta_first_nonjunction(P, a + nld, lim, S.es);
                }
                const unsigned long long len = (unsigned long long)(send - s);
                uint8_t *buf = medp;
                if (len > MED_MAX) {
                    if (tid == 0) {
                        const unsigned long long words = (ENGINE_BYTES(len) + 15) / 16 * 4;
                        unsigned long long off = atomicAdd(&P.st->arena_used, words);
                        if ((off + words) * 4 > P.arena_cap) {
                            atomicExch(&P.st->overflow, 1ull);
                            off = ~0ull;
                        }
                        S.arena_off = off;
                        S.c_giant++;
                        S.c_giant_bytes += len;
                    }
                    __syncthreads();
                    if (S.arena_off == ~0ull) {  // the host re-runs with a larger arena
                        if (tid == 0) S.seg_cnt[i] = 0;
                        __syncthreads();
                        continue;
                    }
                    buf = P.arena + S.arena_off * 4;
                } else if (tid == 0) {
                    S.c_med++;
                }
                EngineMem M;
                M.tok = reinterpret_cast<uint32_t *>(buf);
                M.tok2 = M.tok + len;
                M.pr = reinterpret_cast<uint2 *>(M.tok2 + len);  // 2*len words: 8-B aligned
                M.pr2 = M.pr + len;
                M.sel = reinterpret_cast<uint8_t *>(M.pr2 + len);
                for (unsigned long long j = tid; j < len; j += NT)
                    M.tok[j] = __ldg(&T.base[e != NOSEG ? S.sb[k0 + j] : __ldg(&P.bytes[s + j])]);
                __syncthreads();
                uint32_t passes;
                const uint32_t *res;
                const uint32_t cnt = engine_run(T, M, (uint32_t)len, strict, S.es, &passes, &res);
                if (e != NOSEG)
                    for (uint32_t j = tid; j < cnt; j += NT) S.sid[k0 + j] = res[j];
                if (tid == 0) {
                    S.seg_cnt[i] = cnt;
                    S.c_passes += passes;
                    if (e == NOSEG) {
                        S.ovh_seg = i;
                        S.ovh_src = res;
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
                const unsigned int i = tid * per + j;
                v[j] = i < n_seg ? S.seg_cnt[i] : 0u;
                sum += v[j];
            }
            uint32_t tot;
            uint32_t off = block_excl_sum(sum, S.es, &tot);
#pragma unroll
            for (int j = 0; j < per; ++j) {
                const unsigned int i = tid * per + j;
                if (i < n_seg) S.seg_cnt[i] = off;
                off += v[j];
            }
            if (tid == 0) S.total = tot;
        }
        __syncthreads();
        // ---- decoupled look-back (status words carry the value: relaxed is enough)
        const unsigned long long total = S.total;
        if (wid == 0) {
            const unsigned long long tag = (unsigned long long)P.epoch << 44;
            unsigned long long excl = 0;
            if (t == 0) {
                if (lane == 0) st_relaxed(&P.status[0], tag | (LB_INC << 42) | total);
            } else {
                if (lane == 0) st_relaxed(&P.status[t], tag | (LB_AGG << 42) | total);
                long long pos = (long long)t - 1;
                for (;;) {
                    const long long j = pos - lane;
                    unsigned long long v, flag;
                    if (j >= 0) {
                        do {
                            v = ld_relaxed(&P.status[j]);
                            flag = ((v >> 44) == P.epoch) ? ((v >> 42) & 3ull) : 0ull;
                        } while (flag == 0);
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
                if (lane == 0) st_relaxed(&P.status[t], tag | (LB_INC << 42) | (excl + total));
            }
            if (lane == 0) S.base = excl;
        }
        __syncthreads();
        const unsigned long long base = S.base;
        // ---- store ids
        uint32_t *out = P.out_ids + base;
        const unsigned int oseg = S.ovh_seg;
        for (unsigned int i = tid; i < n_seg; i += NT) {
            if (i == oseg) continue;
            const uint32_t k0 = S.seg_start[i];
            const uint32_t o = S.seg_cnt[i];
            const uint32_t c = (i + 1 < n_seg ? S.seg_cnt[i + 1] : S.total) - o;
            for (uint32_t j = 0; j < c; ++j) out[o + j] = out_id(T, S.sid[k0 + j]);
        }
        if (oseg != 0xFFFFFFFFu) {
            const uint32_t o = S.seg_cnt[oseg];
            const uint32_t c = (oseg + 1 < n_seg ? S.seg_cnt[oseg + 1] : S.total) - o;
            const uint32_t *src = S.ovh_src;
            for (uint32_t j = tid; j < c; j += NT) out[o + j] = out_id(T, src[j]);
        }
        // ---- CSR offsets of documents starting in [a, b) (and at N for the last tile)
        {
            const long long hi = (b == N) ? N + 1 : b;
            for (long long d = d0 + tid; d <= (long long)P.n_docs; d += NT) {
                const long long s = __ldg(&P.doc_offs[d]);
                if (s >= hi) break;
                if (s < a) continue;
                unsigned long long v;
                if (s == N) {
                    v = base + total;
                } else {
                    const int k = (int)(s - a);
                    unsigned int lo = 0, h2 = n_seg;
                    while (lo < h2) {
                        const unsigned int mid = (lo + h2) >> 1;
                        if (S.seg_start[mid] < k) lo = mid + 1; else h2 = mid;
                    }
                    v = base + (lo < n_seg ? S.seg_cnt[lo] : S.total);
                }
                P.out_offs[d] = (long long)v;
            }
        }
        if (tid == 0) {
            EncodeState *st = P.st;
            atomicAdd(&st->n_segments, (unsigned long long)n_seg);
            if (S.c_memo) atomicAdd(&st->memo_hits, (unsigned long long)S.c_memo);
            if (S.c_warp) atomicAdd(&st->short_merges, (unsigned long long)S.c_warp);
            if (S.c_med) atomicAdd(&st->medium_segments, (unsigned long long)S.c_med);
            if (S.c_giant) {
                atomicAdd(&st->giant_segments, (unsigned long long)S.c_giant);
                atomicAdd(&st->giant_bytes, S.c_giant_bytes);
            }
            if (S.c_passes) atomicAdd(&st->engine_passes, (unsigned long long)S.c_passes);
            if (b == N) atomicAdd(&st->n_ids, base + total);
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

cudaError_t launch_encode(const EncodeParams &P, int grid, cudaStream_t s, cudaEvent_t *ev,
                          const cudaAccessPolicyWindow *win) {
    if (ev) cudaEventRecord(ev[0], s);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = sizeof(TileSmem);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    if (win && win->num_bytes) {
        attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[0].val.accessPolicyWindow = *win;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
    }
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_encode, P);
    if (ev) cudaEventRecord(ev[1], s);
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t setup_kernels() {
    return cudaFuncSetAttribute(k_encode, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)sizeof(TileSmem));
}

cudaError_t tile_occupancy(int *blocks) {
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, k_encode, NT, sizeof(TileSmem));
}

cudaError_t launch_lookup(const DevTables &T, const uint32_t *l, const uint32_t *r,
                          unsigned long long n, uint32_t *nw, uint32_t *rank, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_lookup_pairs<<<(unsigned int)((n + 255) / 256), 256, 0, s>>>(T, l, r, n, nw, rank);
    return cudaGetLastError();
}
