// decode.cu -- ids -> bytes on the device.
//
// Restates decode_tokens (/root/reference/pkg/src/lanebpe/byte_codec.py:121-146)
// and Tokenizer.decode (chunker.py:100-101): each id maps to the byte string
// of its vocab symbol; the output is their concatenation; an id outside the
// vocabulary (or whose symbol has a non-byte character) is an error
// (UnknownTokenId).  A batch is a CSR of id sequences; the output is a CSR
// of byte strings.
//
// k_decode: one launch, CTA tiles of TD ids (8 per thread, loaded as uint4 by
// warp-contiguous 512-B rows), lengths from the LUT (L2-resident), warp and
// block scans, a CTA-granular decoupled look-back for the tile's output
// offset, the tile's strings OR-ed into a zeroed shared-memory stage as
// shifted 32-bit words (one 16-B load per string) and stored with 16-B stores
// (tiles whose bytes exceed the stage write directly).  Bound: HBM (4 B read
// per id + its bytes written) once the staging is a few instructions per id.
#include <cuda_runtime.h>

#include <cuda/atomic>

#include "common.cuh"
#include "decode.cuh"

#ifndef GPUBPE_DEC_DT
#define GPUBPE_DEC_DT 512
#endif

namespace {

constexpr int DT = GPUBPE_DEC_DT;      // threads per CTA
constexpr int DPT = 8;               // ids per thread
constexpr int KG = DPT / 4;          // 4-id groups per lane
constexpr int ROW = 32 * DPT;        // ids per warp row
constexpr int TD = DT * DPT;         // ids per tile
constexpr int STAGE = DT * 96;         // staged output bytes per tile (+16 alignment slack)

struct DecSmem {
    uint32_t goff[TD / 4];           // output offset of each 4-id group inside the tile
    uint32_t wsum[DT / 32];
    unsigned long long base, need;
    long long seq_cur;               // first sequence not before the previous tile (tiles of a CTA ascend)
    uint32_t total;
    __align__(16) uint8_t stage[STAGE + 32];
};

// relaxed gpu-scope look-back words (plain PTX, see kernels.cu st_relaxed)
__device__ __forceinline__ void st_rel(unsigned long long *w, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(w), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_rel(unsigned long long *w) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(w) : "memory");
    return v;
}

// id -> (blob offset, length); INF info = unknown id
__device__ __forceinline__ uint32_t info_of(const DecodeParams &P, uint32_t id) {
    return id < P.n_vocab ? __ldg(&P.vinfo[id]) : GPUBPE_INF;
}

// the byte length of a known id from its info word
// (EXT: the vocabulary has empty or >= 255-byte strings; GPT-2 has neither)
template <bool EXT>
__device__ __forceinline__ uint32_t info_len(const DecodeParams &P, uint32_t inf, uint32_t id) {
    const uint32_t l = inf & 0xFFu;
    return EXT && l == LEN_EXT ? __ldg(&P.vlong[id]) : l;
}

}  // namespace

template <bool EXT>
__global__ void __launch_bounds__(DT, 1024 / DT) k_decode(const __grid_constant__ DecodeParams P) {
    extern __shared__ __align__(16) unsigned char dsm_raw[];
    DecSmem &S = *reinterpret_cast<DecSmem *>(dsm_raw);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) S.seq_cur = 0;
    for (;;) {
        if (tid == 0) S.base = atomicAdd(&P.st->tile_ctr, 1ull);
        __syncthreads();
        const unsigned long long t = S.base;
        __syncthreads();
        if (t >= P.n_tiles) break;
        // the stage starts zeroed: strings are OR-ed into it (below)
        for (int q = tid; q < (STAGE + 32) / 16; q += DT) reinterpret_cast<uint4 *>(S.stage)[q] = make_uint4(0, 0, 0, 0);
        const unsigned long long t0 = t * TD;
        // ---- ids: warp row w covers tile ids [w*ROW, (w+1)*ROW); lane l holds
        //      4-id groups g = k*32 + l (k < KG) of that row
        uint32_t id[DPT], len[DPT];
        const unsigned long long row = t0 + (unsigned long long)wid * ROW;
#pragma unroll
        for (int k = 0; k < KG; ++k) {
            const unsigned long long i = row + (unsigned long long)k * 128 + lane * 4;
            if (P.aligned && i + 4 <= P.n_ids) {
                const uint4 v = __ldg(reinterpret_cast<const uint4 *>(P.ids + i));
                id[4 * k] = v.x; id[4 * k + 1] = v.y; id[4 * k + 2] = v.z; id[4 * k + 3] = v.w;
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) id[4 * k + j] = i + j < P.n_ids ? __ldg(&P.ids[i + j]) : 0u;
            }
        }
        uint32_t gs[KG];
#pragma unroll
        for (int k = 0; k < KG; ++k) {
            gs[k] = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const unsigned long long i = row + (unsigned long long)k * 128 + lane * 4 + j;
                uint32_t inf = 0;  // length 0: past the end or unknown
                if (i < P.n_ids) {
                    inf = info_of(P, id[4 * k + j]);
                    if (inf == GPUBPE_INF) {
                        atomicMin(&P.st->bad, i);
                        inf = 0;
                    }
                }
                len[4 * k + j] = inf;  // blob chunk << 8 | length
                gs[k] += inf ? info_len<EXT>(P, inf, id[4 * k + j]) : 0u;
            }
        }
        // ---- offsets: warp scans (k-major), block scan of warp totals
        uint32_t wtot = 0, gex[KG];
#pragma unroll
        for (int k = 0; k < KG; ++k) {
            uint32_t x = gs[k];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(FULL_MASK, x, o);
                if (lane >= o) x += y;
            }
            gex[k] = wtot + x - gs[k];
            wtot += __shfl_sync(FULL_MASK, x, 31);
        }
        if (lane == 31) S.wsum[wid] = wtot;
        __syncthreads();
        if (wid == 0) {
            uint32_t v = lane < DT / 32 ? S.wsum[lane] : 0u;
            uint32_t x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(FULL_MASK, x, o);
                if (lane >= o) x += y;
            }
            if (lane < DT / 32) S.wsum[lane] = x - v;  // exclusive warp offsets
            const uint32_t total = __shfl_sync(FULL_MASK, x, 31);
            // the tile's output offset: precomputed (two-pass mode) or a decoupled
            // look-back over tiles (value+flag+epoch in one word)
            const unsigned long long tag = (unsigned long long)P.epoch << 44;
            unsigned long long excl = 0;
            if (P.tile_base) {
                excl = P.tile_base[t];
            } else if (t == 0) {
                if (lane == 0) st_rel(&P.status[0], tag | (2ull << 42) | total);
            } else {
                if (lane == 0) st_rel(&P.status[t], tag | (1ull << 42) | total);
                long long pos = (long long)t - 1;
                for (;;) {
                    const long long j = pos - lane;
                    unsigned long long v2 = 2ull << 42, flag = 2;
                    if (j >= 0) {
                        for (;;) {
                            v2 = ld_rel(&P.status[j]);
                            flag = ((v2 >> 44) == P.epoch) ? ((v2 >> 42) & 3ull) : 0ull;
                            if (flag) break;
                            __nanosleep(32);
                        }
                    }
                    const unsigned inc = __ballot_sync(FULL_MASK, flag == 2);
                    const int stop = inc ? __ffs(inc) - 1 : 31;
                    unsigned long long val = lane <= stop ? (v2 & ((1ull << 42) - 1)) : 0ull;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(FULL_MASK, val, o);
                    excl += val;
                    if (inc) break;
                    pos -= 32;
                }
                if (lane == 0) st_rel(&P.status[t], tag | (2ull << 42) | (excl + total));
            }
            if (lane == 0) {
                S.base = excl;
                S.total = total;
            }
        }
        __syncthreads();
        const unsigned long long base = S.base;
        const uint32_t total = S.total;
        const uint32_t wbase = S.wsum[wid];
        const bool staged = total <= STAGE;
        const bool fits = base + total <= P.out_cap;
        if (!fits && tid == 0) atomicMax(&P.st->need, base + total);
        // ---- bytes: one 16-B load per id (strings are 16-B aligned and
        //      zero-padded), staged at shift = base & 15 so 16-B chunks of the
        //      stage land on 16-B aligned global addresses
        const uint32_t shift = (uint32_t)(base & 15);
#pragma unroll
        for (int k = 0; k < KG; ++k) {
            uint32_t o = wbase + gex[k];
            S.goff[(wid * KG + k) * 32 + lane] = o;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t inf = len[4 * k + j], l = inf ? info_len<EXT>(P, inf, id[4 * k + j]) : 0u;
                if (l) {
                    const uint4 *src = reinterpret_cast<const uint4 *>(P.blob) + (inf >> 8);
                    if (staged) {  // shared memory (the common case): the zero-padded
                                   // 16-B chunk shifted to its byte offset and OR-ed
                                   // word by word (neighbouring strings share edge words)
                        uint32_t *sw = reinterpret_cast<uint32_t *>(S.stage);
                        for (uint32_t c = 0; c < l; c += 16) {
                            const uint4 v = __ldg(src + (c >> 4));
                            const uint32_t p = shift + o + c, sh = 8 * (p & 3), wi = p >> 2;
                            const uint32_t nw = ((p & 3) + min(16u, l - c) + 3) >> 2;  // words touched
                            atomicOr(&sw[wi], v.x << sh);
                            if (nw > 1) atomicOr(&sw[wi + 1], __funnelshift_l(v.x, v.y, sh));
                            if (nw > 2) atomicOr(&sw[wi + 2], __funnelshift_l(v.y, v.z, sh));
                            if (nw > 3) atomicOr(&sw[wi + 3], __funnelshift_l(v.z, v.w, sh));
                            if (nw > 4) atomicOr(&sw[wi + 4], v.w >> (32 - sh));
                        }
                    } else if (fits) {  // tile larger than the stage: straight to global
                        uint8_t *dst = P.out + base + o;
                        for (uint32_t c = 0; c < l; c += 16) {
                            const uint4 v = __ldg(src + (c >> 4));
                            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
                            const uint32_t m = min(16u, l - c);
                            for (uint32_t b = 0; b < m; ++b) dst[c + b] = (uint8_t)(w[b >> 2] >> (8 * (b & 3)));
                        }
                    }
                }
                o += l;
            }
        }
        __syncthreads();
        // the last warp fixes the sequence offsets while the others store the stage
        const int nstore = P.n_seqs ? DT - 32 : DT;
        if (staged && fits && tid < nstore) {
            // chunk q of the stage covers global [(base & ~15) + 16q, +16)
            const uint32_t end = shift + total, nq = (end + 15) >> 4;
            uint8_t *gdst = P.out + (base & ~15ull);
            for (uint32_t q = tid; q < nq; q += nstore) {
                const uint32_t lo = q * 16, hi = lo + 16;
                if (lo >= shift && hi <= end) {
                    reinterpret_cast<uint4 *>(gdst)[q] = reinterpret_cast<const uint4 *>(S.stage)[q];
                } else {
                    for (uint32_t b = max(lo, shift); b < min(hi, end); ++b) gdst[b] = S.stage[b];
                }
            }
        }
        // ---- byte offsets of the sequences that start in this tile
        if (P.n_seqs && wid == DT / 32 - 1) {
            // first sequence with id_offs >= t0: the 32 after the cursor first, else a
            // 32-ary lower bound beyond them
            long long lo = S.seq_cur, hi = (long long)P.n_seqs;
            {
                const long long idx = lo + lane;
                const bool lt = idx < hi && (unsigned long long)__ldg(&P.id_offs[idx]) < t0;
                const unsigned m = __ballot_sync(FULL_MASK, lt);
                if (m != FULL_MASK) hi = lo = lo + __popc(m);
                else lo += 32;
            }
            while (hi > lo) {
                const long long step = (hi - lo + 31) / 32;
                const long long idx = lo + (long long)lane * step;
                const bool lt = idx < hi && (unsigned long long)__ldg(&P.id_offs[idx]) < t0;
                const unsigned m = __ballot_sync(FULL_MASK, lt);
                if (!m) { hi = lo; break; }
                const int l = 31 - __clz(m);
                lo = lo + (long long)l * step + 1;
                hi = min(hi, lo - 1 + step);
            }
            if (lane == 0) S.seq_cur = lo;
            const bool last_tile = t + 1 == P.n_tiles;
            for (long long d0 = lo;; d0 += 32) {
                const long long d = d0 + lane;
                bool in = false;
                if (d <= (long long)P.n_seqs) {
                    const unsigned long long s = (unsigned long long)__ldg(&P.id_offs[d]);
                    if (s < t0 + TD || last_tile) {
                        in = true;
                        const unsigned long long q = s - t0;  // id index inside the tile
                        unsigned long long v;
                        if (q >= TD || s >= P.n_ids) {
                            v = base + total;
                        } else {
                            const uint32_t w = (uint32_t)(q / ROW), rem = (uint32_t)(q % ROW);
                            const uint32_t k = rem >> 7, l2 = (rem & 127) >> 2, j = rem & 3;
                            uint32_t o = S.goff[(w * KG + k) * 32 + l2];
                            for (uint32_t jj = 0; jj < j; ++jj) {
                                const unsigned long long ii = s - j + jj;
                                const uint32_t iid = __ldg(&P.ids[ii]), inf = info_of(P, iid);
                                o += inf == GPUBPE_INF ? 0u : info_len<EXT>(P, inf, iid);
                            }
                            v = base + o;
                        }
                        P.out_offs[d] = (long long)v;
                    }
                }
                if (__ballot_sync(FULL_MASK, in) != FULL_MASK) break;
            }
        }
        if (t + 1 == P.n_tiles && tid == 0) P.st->n_bytes = base + total;
        __syncthreads();
    }
}

// ---- two-pass mode, second pass: every warp decodes a contiguous range of
//      128-id rows on its own (no CTA barriers).  The row's output offset is the
//      tile's (scanned) plus the bytes of the rows before it in the tile (both
//      from the first pass); lane l holds the row's ids [4l, 4l + 4) and fetches
//      one 16-B record per id -- length and, for strings of up to 15 bytes (all
//      but a few hundred GPT-2 symbols), the string itself -- so an id costs one
//      gather.  The next row's ids are loaded while this one is placed; strings
//      are OR-ed into a warp-private shared-memory stage and stored with 16-B
//      stores (partial edge chunks word/byte-wise: the neighbouring rows belong to
//      other warps).
namespace {
constexpr int RW = 8;                 // warps per CTA
constexpr int RDPT = 4;              // ids per lane
constexpr int RROW = 32 * RDPT;      // ids per row
constexpr int RPT = TD / RROW;       // rows per tile (first-pass row totals)
constexpr int STW = 1024;            // staged bytes per warp (8 per id; larger rows go straight to global)
constexpr int SOFF = 16;             // stage origin (records are placed one byte early)
static_assert(RPT == 32 && TD == 1024 * 4, "row layout matches k_dec_tile_bytes");

__device__ __forceinline__ uint4 load_ids4(const DecodeParams &P, unsigned long long r, int lane) {
    const unsigned long long i = r * RROW + (unsigned long long)lane * RDPT;
    if (P.aligned && i + RDPT <= P.n_ids) return __ldg(reinterpret_cast<const uint4 *>(P.ids + i));
    uint4 v;
    v.x = i < P.n_ids ? __ldg(&P.ids[i]) : 0u;
    v.y = i + 1 < P.n_ids ? __ldg(&P.ids[i + 1]) : 0u;
    v.z = i + 2 < P.n_ids ? __ldg(&P.ids[i + 2]) : 0u;
    v.w = i + 3 < P.n_ids ? __ldg(&P.ids[i + 3]) : 0u;
    return v;
}

__device__ __forceinline__ uint32_t comp(const uint4 &v, int j) {
    return j == 0 ? v.x : j == 1 ? v.y : j == 2 ? v.z : v.w;
}

// OR 16 bytes (v) into the stage at byte position p, touching only the words
// that hold bytes [p, p + n) (32-bit ORs: shared-memory 64-bit ORs measured 1.4x slower)
__device__ __forceinline__ void or16(uint32_t *sw, uint32_t p, const uint4 &v, uint32_t n) {
    const uint32_t sh = 8 * (p & 3), wi = p >> 2, nw = ((p & 3) + n + 3) >> 2;
    atomicOr(&sw[wi], v.x << sh);
    if (nw > 1) atomicOr(&sw[wi + 1], __funnelshift_l(v.x, v.y, sh));
    if (nw > 2) atomicOr(&sw[wi + 2], __funnelshift_l(v.y, v.z, sh));
    if (nw > 3) atomicOr(&sw[wi + 3], __funnelshift_l(v.z, v.w, sh));
    if (nw > 4) atomicOr(&sw[wi + 4], v.w >> (32 - sh));
}

// first index in [lo, hi) whose offset is >= key (offsets ascend), 32-ary
__device__ __forceinline__ long long warp_lower_bound(const long long *a, long long lo, long long hi,
                                                      unsigned long long key, int lane) {
    while (hi > lo) {
        const long long step = (hi - lo + 31) / 32;
        const long long idx = lo + (long long)lane * step;
        const bool lt = idx < hi && (unsigned long long)__ldg(&a[idx]) < key;
        const unsigned m = __ballot_sync(FULL_MASK, lt);
        if (!m) break;
        const int l = 31 - __clz(m);
        lo = lo + (long long)l * step + 1;
        hi = min(hi, lo - 1 + step);
    }
    return lo;
}
}  // namespace

// the byte length in a 16-B record
template <bool EXT>
__device__ __forceinline__ uint32_t rec_len(const uint4 &rec) {
    const uint32_t l = rec.x & 0xFFu;
    return EXT && l == LEN_EXT ? rec.z : l;
}

// the 16-B records of row r's ids (lane's ids [4 lane, 4 lane + 4)); unknown ids
// and ids past the end: length 0 (the first pass reported unknown ones)
__device__ __forceinline__ void load_recs(const DecodeParams &P, unsigned long long r, int lane, const uint4 &idv,
                                          uint4 (&rec)[RDPT]) {
    if ((r + 1) * RROW <= P.n_ids) {  // a full row (warp-uniform): no bounds tests; ids
#pragma unroll                           // >= n_vocab read the zero record at n_vocab
        for (int j = 0; j < RDPT; ++j) rec[j] = __ldg(&P.vrec[min(comp(idv, j), P.n_vocab)]);
        return;
    }
    const unsigned long long i0 = r * RROW + (unsigned long long)lane * RDPT;
#pragma unroll
    for (int j = 0; j < RDPT; ++j) {
        const uint32_t id = comp(idv, j);
        rec[j] = make_uint4(0, 0, 0, 0);
        if (i0 + j < P.n_ids && id < P.n_vocab) rec[j] = __ldg(&P.vrec[id]);
    }
}

struct RowSmem {
    __align__(16) uint8_t stage[RW][SOFF + STW + 48];
};

#ifndef GPUBPE_DEC_MINB
#define GPUBPE_DEC_MINB 4
#endif
template <bool EXT>
__global__ void __launch_bounds__(RW * 32, GPUBPE_DEC_MINB) k_decode_rows(const __grid_constant__ DecodeParams P) {
    extern __shared__ __align__(16) unsigned char rsm_raw[];
    RowSmem &S = *reinterpret_cast<RowSmem *>(rsm_raw);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint8_t *stage = S.stage[wid];
    uint32_t *sw = reinterpret_cast<uint32_t *>(stage);
    for (int q = lane; q < (SOFF + STW + 48) / 16; q += 32) reinterpret_cast<uint4 *>(stage)[q] = make_uint4(0, 0, 0, 0);
    const unsigned long long n_rows = (P.n_ids + RROW - 1) / RROW;
    const unsigned long long gw = (unsigned long long)blockIdx.x * RW + wid, GW = (unsigned long long)gridDim.x * RW;
    const unsigned long long q0 = n_rows / GW, rem = n_rows % GW;
    const unsigned long long r0 = gw * q0 + min(gw, rem), r1 = r0 + q0 + (gw < rem ? 1 : 0);
    if (r0 >= r1) return;
    long long cur = P.n_seqs ? warp_lower_bound(P.id_offs, 0, (long long)P.n_seqs + 1, r0 * RROW, lane) : 0;
    uint4 idv = load_ids4(P, r0, lane);
    unsigned long long next_start = P.n_seqs && cur <= (long long)P.n_seqs ? (unsigned long long)__ldg(&P.id_offs[cur]) : ~0ull;

    // carry_lo >= 0: stage chunk 0 holds the previous row's last, partial 16-B chunk,
    // whose bytes from carry_lo on are ours (the warp's rows are contiguous, so only
    // the range's first and last chunks are shared with other warps)
    int carry_lo = -1;
    __syncwarp();
    for (unsigned long long r = r0; r < r1; ++r) {
        const unsigned long long t = r / RPT;
        const uint32_t rr = (uint32_t)(r % RPT);
        uint32_t pb = lane < (int)rr ? __ldg(&P.row_bytes[t * RPT + lane]) : 0u;
        const unsigned long long tb = __ldg(&P.tile_base[t]);
        uint4 rec[RDPT];
        uint4 nidv = make_uint4(0, 0, 0, 0);
        if (r + 1 < r1) nidv = load_ids4(P, r + 1, lane);
        load_recs(P, r, lane, idv, rec);
        uint32_t sum = 0;
#pragma unroll
        for (int j = 0; j < RDPT; ++j) sum += rec_len<EXT>(rec[j]);
        uint32_t x = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL_MASK, x, o);
            if (lane >= o) x += y;
        }
        const uint32_t excl = x - sum, total = __shfl_sync(FULL_MASK, x, 31);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) pb += __shfl_xor_sync(FULL_MASK, pb, o);
        const unsigned long long base = tb + pb;
        const bool fits = base + total <= P.out_cap;
        if (!fits && lane == 0) atomicMax(&P.st->need, base + total);
        const uint32_t shift = (uint32_t)(base & 15);
        const bool staged = shift + total <= STW;
        if (carry_lo >= 0 && !(staged && fits)) {  // this row is not staged: flush the carried chunk
            uint8_t *gdst = P.out + (base & ~15ull);
            for (uint32_t b = carry_lo + lane; b < shift; b += 32) gdst[b] = stage[SOFF + b];
            __syncwarp();
            if (lane == 0) reinterpret_cast<uint4 *>(stage + SOFF)[0] = make_uint4(0, 0, 0, 0);
            __syncwarp();
            carry_lo = -1;
        }
        const uint32_t own_lo = carry_lo >= 0 ? (uint32_t)carry_lo : shift;
        if (staged) {
            uint32_t o = SOFF + shift + excl;
#pragma unroll
            for (int j = 0; j < RDPT; ++j) {
                const uint32_t l = rec_len<EXT>(rec[j]);
                if (l && l <= 15) {
                    uint4 v = rec[j];
                    v.x &= ~0xFFu;  // the length byte lands (as zero) just before the string
                    or16(sw, o - 1, v, l + 1);
                } else if (l) {
                    const uint4 *src = reinterpret_cast<const uint4 *>(P.blob) + rec[j].y;
                    for (uint32_t c = 0; c < l; c += 16) or16(sw, o + c, __ldg(src + (c >> 4)), min(16u, l - c));
                }
                o += l;
            }
        } else if (fits) {  // more than the stage holds: straight to global, byte by byte
            uint32_t o = excl;
#pragma unroll
            for (int j = 0; j < RDPT; ++j) {
                const uint32_t l = rec_len<EXT>(rec[j]);
                uint8_t *dst = P.out + base + o;
                if (l <= 15) {
                    for (uint32_t b = 0; b < l; ++b) dst[b] = (uint8_t)(comp(rec[j], (b + 1) >> 2) >> (8 * ((b + 1) & 3)));
                } else {
                    const uint8_t *src = P.blob + 16ull * rec[j].y;
                    for (uint32_t b = 0; b < l; ++b) dst[b] = __ldg(src + b);
                }
                o += l;
            }
        }
        __syncwarp();
        const uint32_t end = shift + total, nq = (end + 15) >> 4;
        const bool keep_tail = staged && fits && r + 1 < r1 && (end & 15);
        if (staged && fits) {
            uint8_t *gdst = P.out + (base & ~15ull);
            const uint8_t *sb = stage + SOFF;
            const uint32_t nst = keep_tail ? nq - 1 : nq;  // the partial tail chunk moves on
            for (uint32_t q = lane; q < nst; q += 32) {
                const uint32_t lo = q * 16, hi = lo + 16;
                if (lo >= own_lo && hi <= end) {
                    reinterpret_cast<uint4 *>(gdst)[q] = reinterpret_cast<const uint4 *>(sb)[q];
                } else {  // a chunk shared with another warp's row: bytes, then words, then bytes
                    uint32_t b = max(lo, own_lo);
                    const uint32_t e = min(hi, end);
                    for (; b < e && (b & 3); ++b) gdst[b] = sb[b];
                    for (; b + 4 <= e; b += 4)
                        *reinterpret_cast<uint32_t *>(gdst + b) = *reinterpret_cast<const uint32_t *>(sb + b);
                    for (; b < e; ++b) gdst[b] = sb[b];
                }
                // the lane that stored the chunk clears it (bytes past `end` are never set:
                // records and blob strings are zero-padded)
                reinterpret_cast<uint4 *>(stage + SOFF)[q] = make_uint4(0, 0, 0, 0);
            }
        }
        // byte offsets of the sequences that start in this row (next_start: the
        // first sequence start not yet written, the same in every lane)
        if (P.n_seqs && (next_start < (r + 1) * RROW || r + 1 == n_rows)) {
            const unsigned long long rowlo = r * RROW, rowhi = rowlo + RROW;
            const bool last = r + 1 == n_rows;
            for (;;) {
                const long long d = cur + lane;
                unsigned long long s = ~0ull;
                bool in = false;
                if (d <= (long long)P.n_seqs) {
                    s = (unsigned long long)__ldg(&P.id_offs[d]);
                    in = s < rowhi || last;
                }
                const unsigned long long q = in && s < P.n_ids ? s - rowlo : 0;
                const int src = (int)(q / RDPT) & 31, jj = (int)(q % RDPT);
                uint32_t pre = excl, pick = 0;
#pragma unroll
                for (int j = 0; j < RDPT; ++j) {
                    const uint32_t v = __shfl_sync(FULL_MASK, pre, src);
                    if (j == jj) pick = v;
                    pre += rec_len<EXT>(rec[j]);
                }
                if (in) P.out_offs[d] = (long long)(s >= P.n_ids ? base + total : base + pick);
                const unsigned m = __ballot_sync(FULL_MASK, in);
                cur += __popc(m);
                if (m != FULL_MASK) break;
            }
            next_start = cur <= (long long)P.n_seqs ? (unsigned long long)__ldg(&P.id_offs[cur]) : ~0ull;
        }
        if (r + 1 == n_rows && lane == 0) P.st->n_bytes = base + total;
        __syncwarp();
        if (staged && !fits)  // staged but not stored (the call fails with the size needed)
            for (uint32_t q = lane; q < nq; q += 32) reinterpret_cast<uint4 *>(stage + SOFF)[q] = make_uint4(0, 0, 0, 0);
        if (keep_tail) {  // lane 0 moves the unstored tail chunk to the front
            if (lane == 0) {
                uint4 *c = reinterpret_cast<uint4 *>(stage + SOFF);
                const uint4 tail = c[nq - 1];
                c[nq - 1] = make_uint4(0, 0, 0, 0);
                c[0] = tail;
            }
            carry_lo = nq == 1 ? (int)own_lo : 0;
        } else {
            carry_lo = -1;
        }
        __syncwarp();
        idv = nidv;
    }
}

cudaError_t decode_rows_occupancy(int *blocks) {
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, k_decode_rows<false>, RW * 32, sizeof(RowSmem));
}

cudaError_t launch_decode_rows(const DecodeParams &P, int grid, cudaStream_t s) {
    if (P.ext) k_decode_rows<true><<<grid, RW * 32, sizeof(RowSmem), s>>>(P);
    else k_decode_rows<false><<<grid, RW * 32, sizeof(RowSmem), s>>>(P);
    return cudaGetLastError();
}

// ---- two-pass mode: tile byte totals (one CTA per tile, every CTA at once),
//      then one CTA scans them into tile offsets; k_decode then needs no look-back
template <bool EXT>
__global__ void __launch_bounds__(256) k_dec_tile_bytes(const __grid_constant__ DecodeParams P,
                                                        unsigned long long *tile_bytes) {
    constexpr int IT = TD / (256 * 4);  // 4-id groups per thread, all loads issued together
    __shared__ uint32_t red[8];
    const unsigned long long t = blockIdx.x, t0 = t * TD;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t id[IT][4];
#pragma unroll
    for (int k = 0; k < IT; ++k) {
        const unsigned long long i = t0 + (unsigned long long)k * 1024 + threadIdx.x * 4;
        if (P.aligned && i + 4 <= P.n_ids) {
            const uint4 v = __ldg(reinterpret_cast<const uint4 *>(P.ids + i));
            id[k][0] = v.x; id[k][1] = v.y; id[k][2] = v.z; id[k][3] = v.w;
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) id[k][j] = i + j < P.n_ids ? __ldg(&P.ids[i + j]) : 0u;
        }
    }
    // lengths from the 1-byte table (128 ids per L1 line: the frequent low ids share lines)
    uint32_t tot = 0;
#pragma unroll
    for (int k = 0; k < IT; ++k) {
        const unsigned long long i = t0 + (unsigned long long)k * 1024 + threadIdx.x * 4;
        uint32_t sk = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (i + j < P.n_ids) {
                uint32_t l = id[k][j] < P.n_vocab ? __ldg(&P.vlen[id[k][j]]) : 0u;
                if (l == 0) atomicMin(&P.st->bad, i + j);
                if (EXT && l == LEN_EXT) l = __ldg(&P.vlong[id[k][j]]);
                sk += l;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sk += __shfl_xor_sync(FULL_MASK, sk, o);
        // warp w at k covers ids [k*1024 + w*128, +128): row 8k + w of the tile
        if (P.row_bytes && lane == 0) P.row_bytes[t * (TD / 128) + 8 * k + wid] = sk;
        tot += sk;
    }
    if (lane == 0) red[wid] = tot;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int w = 0; w < 8; ++w) s += red[w];
        tile_bytes[t] = s;
    }
}

// one CTA: exclusive scan of the tile byte totals.  Up to SCAN_SMEM tiles (117 M
// ids) the totals are staged in shared memory by coalesced loads, each thread
// scans a contiguous run there and the bases leave by coalesced stores; larger
// batches scan in global memory directly.
constexpr unsigned SCAN_SMEM = 28 << 10;  // tiles (224 KiB of u64)
__global__ void __launch_bounds__(1024) k_dec_scan(const unsigned long long *tile_bytes, unsigned long long n,
                                                   unsigned long long *tile_base) {
    extern __shared__ unsigned long long sscan[];
    __shared__ unsigned long long wsum[32];
    const bool staged = n <= SCAN_SMEM;
    if (staged)
        for (unsigned long long i = threadIdx.x; i < n; i += 1024) sscan[i] = __ldg(&tile_bytes[i]);
    __syncthreads();
    const unsigned long long *src = staged ? sscan : tile_bytes;
    unsigned long long *dst = staged ? sscan : tile_base;
    const unsigned long long per = (n + 1023) / 1024, lo = min(n, threadIdx.x * per), hi = min(n, lo + per);
    unsigned long long s = 0;
    for (unsigned long long i = lo; i < hi; ++i) s += src[i];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned long long x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(FULL_MASK, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    if (wid == 0) {
        unsigned long long v = wsum[lane], y2 = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(FULL_MASK, y2, o);
            if (lane >= o) y2 += y;
        }
        wsum[lane] = y2 - v;
    }
    __syncthreads();
    unsigned long long run = wsum[wid] + x - s;
    for (unsigned long long i = lo; i < hi; ++i) {
        const unsigned long long t = src[i];
        dst[i] = run;
        run += t;
    }
    if (staged) {
        __syncthreads();
        for (unsigned long long i = threadIdx.x; i < n; i += 1024) tile_base[i] = sscan[i];
    }
}

cudaError_t launch_decode_offsets(const DecodeParams &P, unsigned long long *tile_bytes,
                                  unsigned long long *tile_base, cudaStream_t s) {
    if (P.n_tiles == 0) return cudaSuccess;
    if (P.ext) k_dec_tile_bytes<true><<<(unsigned int)P.n_tiles, 256, 0, s>>>(P, tile_bytes);
    else k_dec_tile_bytes<false><<<(unsigned int)P.n_tiles, 256, 0, s>>>(P, tile_bytes);
    const size_t sm = P.n_tiles <= SCAN_SMEM ? P.n_tiles * sizeof(unsigned long long) : 0;
    k_dec_scan<<<1, 1024, sm, s>>>(tile_bytes, P.n_tiles, tile_base);
    return cudaGetLastError();
}

size_t decode_smem_bytes() { return sizeof(DecSmem); }
int decode_tile_ids() { return TD; }

cudaError_t setup_decode() {
    cudaError_t e = cudaFuncSetAttribute(k_decode<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(DecSmem));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_decode<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(DecSmem));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_dec_scan, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(SCAN_SMEM * sizeof(unsigned long long)));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_decode_rows<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(RowSmem));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_decode_rows<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(RowSmem));
}

cudaError_t decode_occupancy(int *blocks) {
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, k_decode<false>, DT, sizeof(DecSmem));
}

cudaError_t launch_decode(const DecodeParams &P, int grid, cudaStream_t s) {
    if (P.ext) k_decode<true><<<grid, DT, sizeof(DecSmem), s>>>(P);
    else k_decode<false><<<grid, DT, sizeof(DecSmem), s>>>(P);
    return cudaGetLastError();
}
