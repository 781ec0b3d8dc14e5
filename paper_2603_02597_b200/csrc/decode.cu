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

__device__ __forceinline__ void st_rel(unsigned long long *w, unsigned long long v) {
    cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> r(*w);
    r.store(v, cuda::memory_order_relaxed);
}
__device__ __forceinline__ unsigned long long ld_rel(unsigned long long *w) {
    cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> r(*w);
    return r.load(cuda::memory_order_relaxed);
}

// id -> (blob offset, length); INF info = unknown id
__device__ __forceinline__ uint32_t info_of(const DecodeParams &P, uint32_t id) {
    return id < P.n_vocab ? __ldg(&P.vinfo[id]) : GPUBPE_INF;
}

}  // namespace

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
                gs[k] += inf & 0xFFu;
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
                const uint32_t inf = len[4 * k + j], l = inf & 0xFFu;
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
                                const uint32_t inf = info_of(P, __ldg(&P.ids[ii]));
                                o += inf == GPUBPE_INF ? 0u : (inf & 0xFFu);
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

// ---- two-pass mode: tile byte totals (one CTA per tile, every CTA at once),
//      then one CTA scans them into tile offsets; k_decode then needs no look-back
__global__ void __launch_bounds__(256) k_dec_tile_bytes(const __grid_constant__ DecodeParams P,
                                                        unsigned long long *tile_bytes) {
    __shared__ unsigned long long red[8];
    const unsigned long long t = blockIdx.x, t0 = t * TD;
    constexpr int IT = TD / (256 * 4);  // 4-id groups per thread, all loads issued together
    unsigned long long sum = 0;
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
#pragma unroll
    for (int k = 0; k < IT; ++k) {
        const unsigned long long i = t0 + (unsigned long long)k * 1024 + threadIdx.x * 4;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (i + j < P.n_ids) {
                const uint32_t inf = info_of(P, id[k][j]);
                if (inf == GPUBPE_INF) atomicMin(&P.st->bad, i + j);
                else sum += inf & 0xFFu;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(FULL_MASK, sum, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int w = 0; w < 8; ++w) s += red[w];
        tile_bytes[t] = s;
    }
}

__global__ void __launch_bounds__(1024) k_dec_scan(const unsigned long long *tile_bytes, unsigned long long n,
                                                   unsigned long long *tile_base) {
    __shared__ unsigned long long wsum[32];
    const unsigned long long per = (n + 1023) / 1024, lo = min(n, threadIdx.x * per), hi = min(n, lo + per);
    unsigned long long s = 0;
    for (unsigned long long i = lo; i < hi; ++i) s += tile_bytes[i];
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
        tile_base[i] = run;
        run += tile_bytes[i];
    }
}

cudaError_t launch_decode_offsets(const DecodeParams &P, unsigned long long *tile_bytes,
                                  unsigned long long *tile_base, cudaStream_t s) {
    if (P.n_tiles == 0) return cudaSuccess;
    k_dec_tile_bytes<<<(unsigned int)P.n_tiles, 256, 0, s>>>(P, tile_bytes);
    k_dec_scan<<<1, 1024, 0, s>>>(tile_bytes, P.n_tiles, tile_base);
    return cudaGetLastError();
}

size_t decode_smem_bytes() { return sizeof(DecSmem); }
int decode_tile_ids() { return TD; }

cudaError_t setup_decode() {
    return cudaFuncSetAttribute(k_decode, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(DecSmem));
}

cudaError_t decode_occupancy(int *blocks) {
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, k_decode, DT, sizeof(DecSmem));
}

cudaError_t launch_decode(const DecodeParams &P, int grid, cudaStream_t s) {
    k_decode<<<grid, DT, sizeof(DecSmem), s>>>(P);
    return cudaGetLastError();
}
