// pretok.cu -- optional GPT-2 regex pre-tokenization on the device
// (never the default: the reference has none,
// SPEC.md:93,95).
//
// tiktoken's GPT-2 pattern
//   '(?:[sdmt]|ll|ve|re)| ?\p{L}+| ?\p{N}+| ?[^\s\p{L}\p{N}]+|\s+(?!\S)|\s+
// splits text into pre-tokens that BPE never merges across.  Its token starts
// are decidable from a few neighbouring code points (classes L, N, S = \s,
// O = other; ' ' and '\'' and the contraction letters by value), which makes
// them one more set of exact cut points for k_encode:
//   start of text                                   boundary
//   cur \s:     prev not \s                         boundary (a whitespace run starts)
//               prev \s, next exists and is not \s  boundary (the run's last char splits off)
//   cur not \s: prev \s                             boundary iff prev != ' ' (a space joins
//                                                   the following token)
//               prev is an apostrophe starting a
//               contraction ('s 'd 'm 't 'll 've 're) no boundary inside it, boundary after
//               otherwise                           boundary iff the class changes
// where an apostrophe starts a contraction iff it is at a token start (text
// start, or prev in L/N, or prev \s other than ' ').  The rules are checked
// against the regex itself in tests (and reproduce tiktoken's ids there).
//
// k_pretok: one thread per 32-byte word of the batch; bit k of word w =
// token start before byte 32w + k.  Code points: a byte that is not
// 10xxxxxx starts one (invalid sequences become single "other" code points;
// stray continuation bytes join the preceding one).  Document starts are
// text starts.
//
// Common case (the word lies in one document and its 48-byte window
// [32w - 8, 32w + 40) is ASCII there): code points are bytes, and the rules
// are evaluated bit-parallel on 48-bit masks (bit j = byte 32w - 8 + j) built
// with SWAR byte-range tests; the word's bytes arrive in two coalesced 16-B
// loads and the context bytes from the neighbouring lanes by shuffle.
// Otherwise a per-code-point scalar path decodes UTF-8 around the word.
#include <cuda_runtime.h>

#include "common.cuh"
#include "pretok.cuh"

namespace {

constexpr int PT = 256;      // threads per CTA
constexpr int BACK = 24;     // bytes decoded before a word (>= 4 code points of context)
constexpr int AHEAD = 12;    // bytes decoded after it (2 code points of lookahead)
#ifndef GPUBPE_PRETOK_PW
#define GPUBPE_PRETOK_PW 2
#endif
constexpr int PW = GPUBPE_PRETOK_PW;  // words per thread

enum : uint8_t { C_O = 0, C_L = 1, C_N = 2, C_S = 3 };

__device__ __forceinline__ uint8_t cp_class(const PretokParams &Q, uint32_t cp) {
    if (cp >= Q.n_cps) return C_O;
    return (uint8_t)((__ldg(&Q.classes[cp >> 2]) >> (2 * (cp & 3))) & 3u);
}

constexpr unsigned long long K1 = 0x0101010101010101ull, K80 = 0x8080808080808080ull;

// 0x80 in every byte of x whose value lies in [lo, hi] (values < 0x80; x7 = x & 0x7F.., hb = x & 0x80..)
__device__ __forceinline__ unsigned long long in_range(unsigned long long x7, unsigned long long hb,
                                                       unsigned lo, unsigned hi) {
    const unsigned long long ge = x7 + (0x80ull - lo) * K1;  // bit 7 set iff v >= lo (no carry out of a byte)
    const unsigned long long gt = x7 + (0x7Full - hi) * K1;  // bit 7 set iff v > hi
    return ge & ~gt & ~hb & K80;
}

// bit k = bit 7 of byte k (m has only bits 7 of its bytes set)
__device__ __forceinline__ unsigned movemask8(unsigned long long m) {
    return (unsigned)(((m >> 7) * 0x0102040810204080ull) >> 56);
}

struct Masks {
    unsigned long long L, N, S, SP, AP, NA;
};

__device__ __forceinline__ Masks build_masks(const unsigned long long (&win)[6]) {
    Masks M{0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        const unsigned long long x = win[k], hb = x & K80, x7 = x & ~K80;
        const unsigned long long sp = in_range(x7, hb, ' ', ' ');
        M.L |= (unsigned long long)movemask8(in_range(x7 | 0x20 * K1, hb, 'a', 'z')) << (8 * k);
        M.N |= (unsigned long long)movemask8(in_range(x7, hb, '0', '9')) << (8 * k);
        M.S |= (unsigned long long)movemask8(in_range(x7, hb, 9, 13) | sp) << (8 * k);
        M.SP |= (unsigned long long)movemask8(sp) << (8 * k);
        M.AP |= (unsigned long long)movemask8(in_range(x7, hb, '\'', '\'')) << (8 * k);
        M.NA |= (unsigned long long)movemask8(hb) << (8 * k);
    }
    return M;
}

__device__ __forceinline__ unsigned long long eq_mask(const unsigned long long (&win)[6], unsigned c) {
    unsigned long long m = 0;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        const unsigned long long x = win[k], hb = x & K80;
        m |= (unsigned long long)movemask8(in_range(x & ~K80, hb, c, c)) << (8 * k);
    }
    return m;
}

// Token-start bits of the 32 positions j in [8, 40) of the window (bit j:
// byte 32w - 8 + j), E = bytes of the word's document.  The class masks hold,
// at every byte, the class of the code point containing it; LEAD marks code
// point starts and NNS, at a start, "the next code point exists and is not
// \s".  For ASCII every byte is a code point (LEAD = E, NNS = (E & ~S) >> 1).
__device__ __forceinline__ uint32_t rules_bitparallel(const unsigned long long (&win)[6], const Masks &M0,
                                                      unsigned long long E, unsigned long long LEAD,
                                                      unsigned long long NNS) {
    const unsigned long long L = M0.L & E, N = M0.N & E, S = M0.S & E, SP = M0.SP & E, AP = M0.AP & E;
    unsigned long long C2 = 0, C3 = 0;  // contractions starting at j: 's 'd 'm 't / 'll 've 're
    if (AP) {
        // an apostrophe starts one iff it is at a token start: text start, or prev in L/N, or prev \s other than ' '
        const unsigned long long TS = ~(E << 1) | ((L | N | (S & ~SP)) << 1);
        const unsigned long long a = AP & TS;
        const unsigned long long sdmt = (eq_mask(win, 's') | eq_mask(win, 'd') | eq_mask(win, 'm') |
                                         eq_mask(win, 't')) & E;
        const unsigned long long l = eq_mask(win, 'l') & E, e = eq_mask(win, 'e') & E;
        const unsigned long long vr = (eq_mask(win, 'v') | eq_mask(win, 'r')) & E;
        C2 = a & (sdmt >> 1);
        C3 = a & (((l >> 1) & (l >> 2)) | ((vr >> 1) & (e >> 2)));
    }
    const unsigned long long C = C2 | C3;
    const unsigned long long B =
        ~(E << 1)                                                    // text start
        | (S & (~(S << 1) | NNS))                                    // whitespace run start / last char of a run
        | (~S & (S << 1) & ~(SP << 1))                               // after \s other than ' '
        | (~S & ~(S << 1) & ~((C << 1) | (C3 << 2)) &                // not inside a contraction:
           ((C2 << 2) | (C3 << 3) | (L ^ (L << 1)) | (N ^ (N << 1))));  // after one, or a class change
    return (uint32_t)((B & E & LEAD) >> 8);
}

// bytes j .. j + 3 of the window (little endian), 0 <= j < 44
__device__ __forceinline__ uint32_t win_bytes4(const unsigned long long (&win)[6], int j) {
    unsigned long long lo = 0, hi = 0;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        if (k == (j >> 3)) lo = win[k];
        if (k == (j >> 3) + 1) hi = win[k];
    }
    const int sh = 8 * (j & 7);
    return (uint32_t)(sh ? (lo >> sh) | (hi << (64 - sh)) : lo);
}

// Masks of a window with non-ASCII bytes (the scalar path's code point rules:
// a byte that is not 10xxxxxx starts a code point, as does the document's
// first byte; a sequence whose continuation run does not match its lead byte
// is one "other" code point).  Returns false when a continuation run longer
// than 3 bytes (a code point the window cannot hold) calls for the scalar path.
__device__ __forceinline__ bool unicode_masks(const PretokParams &Q, const unsigned long long (&win)[6], Masks &M,
                                              unsigned long long E, int jlo, unsigned long long &LEAD,
                                              unsigned long long &NNS) {
    unsigned long long CONT = 0;
#pragma unroll
    for (int k = 0; k < 6; ++k) CONT |= (unsigned long long)movemask8(win[k] & ~(win[k] << 1) & K80) << (8 * k);
    const unsigned long long start = jlo >= 0 ? (1ull << jlo) : 0ull;  // the document's first byte
    LEAD = (~CONT | start) & E;
    const unsigned long long CE = CONT & E & ~start;  // continuation bytes joined to the preceding start
    if (CE & (CE << 1) & (CE << 2) & (CE << 3)) return false;
    // non-ASCII starts below 44 (the next code point of byte 39's) get their class from the table
    for (unsigned long long nl = LEAD & M.NA & ((1ull << 44) - 1); nl; nl &= nl - 1) {
        const int j = __ffsll((long long)nl) - 1;
        const uint32_t x = win_bytes4(win, j), b0 = x & 0xFFu;
        const int need = b0 >= 0xF0u ? 3 : b0 >= 0xE0u ? 2 : b0 >= 0xC0u ? 1 : -1;
        const unsigned long long after = CE >> (j + 1);
        const int run = (after & 1) ? ((after & 2) ? ((after & 4) ? 3 : 2) : 1) : 0;
        uint8_t c = C_O;
        if (need > 0 && run == need && b0 < 0xF8u) {
            uint32_t cp = b0 & (0x3Fu >> need);
            for (int k = 1; k <= need; ++k) cp = (cp << 6) | ((x >> (8 * k)) & 0x3Fu);
            c = cp_class(Q, cp);
        }
        const unsigned long long bit = 1ull << j;
        if (c == C_L) M.L |= bit;
        else if (c == C_N) M.N |= bit;
        else if (c == C_S) M.S |= bit;
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {  // every byte of a code point carries its class
        M.L |= (M.L << 1) & CE;
        M.N |= (M.N << 1) & CE;
        M.S |= (M.S << 1) & CE;
    }
    NNS = (LEAD & ~M.S) >> 1;  // at a code point's last byte: the next one exists and is not \s
#pragma unroll
    for (int k = 0; k < 3; ++k) NNS |= (NNS >> 1) & (CE >> 1);  // ... carried back to its start
    return true;
}

// SWAR forms on 4 bytes: 0x80 in each byte whose value is in [lo, hi]
// (x7 = x & 0x7F.., nh = ~x & 0x80.., so bytes >= 0x80 never match)
__device__ __forceinline__ uint32_t rng4(uint32_t x7, uint32_t nh, uint32_t lo, uint32_t hi) {
    return (x7 + (0x80u - lo) * 0x01010101u) & ~(x7 + (0x7Fu - hi) * 0x01010101u) & nh;
}
__device__ __forceinline__ uint32_t movemask4(uint32_t m) { return (((m >> 7) * 0x00204081u) >> 21) & 0xFu; }

// Token-start bits of the word when bytes [p0 - 4, p0 + 36) all lie in its
// document, are ASCII and hold no apostrophe: the rules without the
// contraction terms, evaluated on bytes in place (bit 7 of each byte) with
// funnel shifts for the neighbouring positions; x[i] = bytes p0 - 4 + 4i.
__device__ __forceinline__ uint32_t rules_swar(const uint32_t (&x)[10]) {
    uint32_t L[10], N[10], S[10], SP[10];
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        const uint32_t x7 = x[i] & 0x7F7F7F7Fu, nh = ~x[i] & 0x80808080u;
        L[i] = rng4(x7 | 0x20202020u, nh, 'a', 'z');
        N[i] = rng4(x7, nh, '0', '9');
        SP[i] = rng4(x7, nh, ' ', ' ');
        S[i] = rng4(x7, nh, 9, 13) | SP[i];
    }
    uint32_t bits = 0;
#pragma unroll
    for (int i = 1; i < 9; ++i) {
        const uint32_t pS = __funnelshift_l(S[i - 1], S[i], 8), nS = __funnelshift_r(S[i], S[i + 1], 8);
        const uint32_t pSP = __funnelshift_l(SP[i - 1], SP[i], 8);
        const uint32_t pL = __funnelshift_l(L[i - 1], L[i], 8), pN = __funnelshift_l(N[i - 1], N[i], 8);
        const uint32_t B = (S[i] & (~pS | ~nS)) | (~S[i] & pS & ~pSP) | (~S[i] & ~pS & ((L[i] ^ pL) | (N[i] ^ pN)));
        bits |= movemask4(B & 0x80808080u) << (4 * (i - 1));
    }
    return bits;
}

// Token-start bits of the word [p0, p1) of documents d.. from its 48-byte
// window: the SWAR path, the bit-parallel mask paths, else the scalar code
// point path.
__device__ __forceinline__ uint32_t word_bits(const PretokParams &Q, const uint8_t *sasc, long long p0,
                                              long long p1, const unsigned long long (&win)[6], long long d) {
    if (Q.ascii_std) {
        const long long ds = __ldg(&Q.doc_offs[d]), de = __ldg(&Q.doc_offs[d + 1]);
        if ((Q.paths & 1) && ds <= p0 - 4 && de >= p0 + 36) {
            uint32_t x[10], hb = 0, ap = 0;
#pragma unroll
            for (int i = 0; i < 10; ++i) {
                const int b = 4 + 4 * i;  // byte offset in the 48-byte window
                x[i] = (uint32_t)(win[b >> 3] >> (8 * (b & 7)));
                hb |= x[i];
                ap |= rng4(x[i] & 0x7F7F7F7Fu, ~x[i] & 0x80808080u, '\'', '\'');
            }
            if (((hb & 0x80808080u) | ap) == 0) return rules_swar(x);
        }
        // every document meeting [p0, p1) in turn, on the bit-parallel masks restricted to it
        const Masks M = build_masks(win);
        uint32_t bits = 0;
        bool ok = true;
        for (long long dd = d;; ++dd) {
            const long long s0 = __ldg(&Q.doc_offs[dd]), s1 = __ldg(&Q.doc_offs[dd + 1]);
            if (s0 >= p1) break;
            const long long jlo = max(0ll, s0 - (p0 - 8)), jhi = min(48ll, s1 - (p0 - 8));
            if (jhi > jlo) {
                const unsigned long long E = ((1ull << jhi) - 1) & ~((1ull << jlo) - 1);
                if (M.NA & E) {
                    // non-ASCII bytes in this document's part of the window
                    Masks MU = M;
                    unsigned long long LEAD, NNS;
                    const int start = s0 >= p0 - 8 ? (int)jlo : -1;  // document start inside the window
                    if (!(Q.paths & 4) || !unicode_masks(Q, win, MU, E, start, LEAD, NNS)) {
                        ok = false;
                        break;
                    }
                    bits |= rules_bitparallel(win, MU, E, LEAD, NNS);
                } else if (Q.paths & 2) {
                    bits |= rules_bitparallel(win, M, E, E, (E & ~M.S) >> 1);
                } else {
                    ok = false;
                    break;
                }
            }
            if (s1 >= p1) break;
        }
        if (ok) return bits;
    }
    uint32_t bits = 0;
    for (long long pos = p0; pos < p1;) {
        while (__ldg(&Q.doc_offs[d + 1]) <= pos) ++d;  // skip empty documents
        const long long ds = __ldg(&Q.doc_offs[d]), de = __ldg(&Q.doc_offs[d + 1]);
        const long long seg_end = min(p1, de);
        // the code points of [q, min(de, seg_end + AHEAD)) of this document, streamed
        // through a register window: slot 4 = code point k (the one decided), slots
        // 0-3 = k-4 .. k-1, slot 5 = k+1 (v5: it exists)
        long long q = max(ds, pos - BACK);
        while (q > ds && q < pos && (__ldg(&Q.bytes[q]) & 0xC0u) == 0x80u) ++q;
        const long long qe = min(de, seg_end + AHEAD);
        const bool text_start = q == ds;  // code point 0 is the document's first
        uint8_t C[6] = {0, 0, 0, 0, 0, 0}, A[6] = {0, 0, 0, 0, 0, 0};
        long long P4 = 0, P5 = 0, i = q;
        bool v5 = false;
        auto next_cp = [&]() {  // decode the code point at byte i into slot 5
            v5 = i < qe;
            if (!v5) return;
            const uint32_t b0 = __ldg(&Q.bytes[i]);
            long long j = i + 1;
            while (j < de && (__ldg(&Q.bytes[j]) & 0xC0u) == 0x80u) ++j;  // continuation bytes join
            uint8_t c = C_O, a = 0;
            if (b0 < 0x80u) {
                c = sasc[b0];
                a = (uint8_t)b0;
            } else {
                const int need = b0 >= 0xF0u ? 3 : b0 >= 0xE0u ? 2 : b0 >= 0xC0u ? 1 : -1;
                if (need > 0 && j - i == need + 1 && b0 < 0xF8u) {
                    uint32_t cp = b0 & (0x3Fu >> need);
                    for (int k = 1; k <= need; ++k) cp = (cp << 6) | (__ldg(&Q.bytes[i + k]) & 0x3Fu);
                    c = cp_class(Q, cp);
                }
            }
            C[5] = c;
            A[5] = a;
            P5 = i;
            i = j;
        };
        next_cp();
        for (long long k = 0; v5; ++k) {
#pragma unroll
            for (int t = 0; t < 5; ++t) {
                C[t] = C[t + 1];
                A[t] = A[t + 1];
            }
            P4 = P5;
            next_cp();
            if (P4 >= seg_end) break;
            if (P4 < pos) continue;
            // token start before code point j (in slot s): the apostrophe test
            auto tstart = [&](long long j, int s) -> bool {
                if (j == 0) return text_start;
                return C[s - 1] == C_L || C[s - 1] == C_N || (C[s - 1] == C_S && A[s - 1] != ' ');
            };
            auto clen = [&](long long j, int s) -> int {  // contraction at code point j: its length, else 0
                if (j < 0 || A[s] != '\'' || !tstart(j, s)) return 0;
                const uint8_t a = (s + 1 < 5 || v5) ? A[s + 1] : 0, b = (s + 2 < 5 || v5) ? A[s + 2] : 0;
                if (a == 's' || a == 'd' || a == 'm' || a == 't') return 2;
                if ((a == 'l' && b == 'l') || (a == 'v' && b == 'e') || (a == 'r' && b == 'e')) return 3;
                return 0;
            };
            bool b;
            if (k == 0) {
                b = text_start;  // (a word never starts BACK bytes into a document's interior)
            } else if (C[4] == C_S) {
                b = C[3] != C_S || (v5 && C[5] != C_S);
            } else if (C[3] == C_S) {
                b = A[3] != ' ';
            } else if (clen(k - 1, 3)) {
                b = false;
            } else if (clen(k - 2, 2) == 3) {
                b = false;
            } else if (clen(k - 2, 2) == 2 || clen(k - 3, 1) == 3) {
                b = true;
            } else {
                b = C[4] != C[3];
            }
            if (b) bits |= 1u << (uint32_t)(P4 - p0);
        }
        pos = seg_end;
    }
    return bits;
}

// The 32 bytes [p0, p0 + 32) as four little-endian words (0 past n), and for
// lanes 0 / 31 the 8 bytes before / after them (the warp's window edges).
__device__ __forceinline__ void load_word(const PretokParams &Q, long long p0, bool active, int lane,
                                          unsigned long long (&r)[4], unsigned long long &edge) {
    const long long n = (long long)Q.n_bytes;
    const bool aligned = ((reinterpret_cast<uintptr_t>(Q.bytes) & 15) == 0);
    if (active && aligned && p0 + 32 <= n) {
        const uint4 *src = reinterpret_cast<const uint4 *>(Q.bytes + p0);
        const uint4 u = __ldg(src), v = __ldg(src + 1);
        r[0] = ((unsigned long long)u.y << 32) | u.x;
        r[1] = ((unsigned long long)u.w << 32) | u.z;
        r[2] = ((unsigned long long)v.y << 32) | v.x;
        r[3] = ((unsigned long long)v.w << 32) | v.z;
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            unsigned long long x = 0;
            for (int b = 7; b >= 0; --b) {
                const long long p = p0 + 8 * k + b;
                x = (x << 8) | ((active && p < n) ? __ldg(&Q.bytes[p]) : 0u);
            }
            r[k] = x;
        }
    }
    edge = 0;
    if (lane == 0 || lane == 31) {
        const long long q = lane == 0 ? p0 - 8 : p0 + 32;
        if (aligned && q >= 0 && q + 8 <= n) {
            edge = __ldg(reinterpret_cast<const unsigned long long *>(Q.bytes + q));
        } else {
            for (int b = 7; b >= 0; --b) {
                const long long p = q + b;
                edge = (edge << 8) | ((active && p >= 0 && p < n) ? __ldg(&Q.bytes[p]) : 0u);
            }
        }
    }
}

}  // namespace

#ifndef GPUBPE_PRETOK_MINB
#define GPUBPE_PRETOK_MINB 4
#endif
// PW words per thread: word k of thread t is the CTA's word k * PT + t (coalesced
// rows); every word's bytes are loaded before the document search and the barrier.
__global__ void __launch_bounds__(PT, GPUBPE_PRETOK_MINB) k_pretok(const __grid_constant__ PretokParams Q) {
    __shared__ uint8_t sasc[128];
    __shared__ long long sdoc[2];  // documents holding the CTA's first and last byte
    const int lane = threadIdx.x & 31;
    const unsigned long long w0 = (unsigned long long)blockIdx.x * (PT * PW) + threadIdx.x;
    unsigned long long r[PW][4], edge[PW];
#pragma unroll
    for (int k = 0; k < PW; ++k)
        load_word(Q, (long long)(w0 + k * PT) * 32, w0 + k * PT < Q.n_words, lane, r[k], edge[k]);
    if (threadIdx.x < 128) sasc[threadIdx.x] = Q.ascii[threadIdx.x];
    if (threadIdx.x < 64) {  // warps 0 / 1: 32-ary searches for the CTA's first / last byte
        const int wsel = threadIdx.x >> 5, ln = threadIdx.x & 31;
        const long long nb = (long long)Q.n_bytes;
        const long long q =
            min(nb - 1, ((long long)blockIdx.x * PT * PW + (wsel ? PT * PW - 1 : 0)) * 32 + (wsel ? 31 : 0));
        long long lo = 0, hi = (long long)Q.n_docs - 1;  // last d in [lo, hi] with offs[d] <= q
        while (hi > lo) {
            const long long step = (hi - lo + 32) / 32;
            const long long idx = lo + (long long)ln * step;
            const bool ok = idx <= hi && __ldg(&Q.doc_offs[idx]) <= q;
            const unsigned m = __ballot_sync(FULL_MASK, ok);  // lane 0 always holds
            lo = lo + (long long)(31 - __clz(m)) * step;
            hi = min(hi, lo + step - 1);
        }
        if (ln == 0) sdoc[wsel] = lo;
    }
    __syncthreads();
    const long long n = (long long)Q.n_bytes;
    long long d = sdoc[0];
    const long long dhi = sdoc[1];
#pragma unroll
    for (int k = 0; k < PW; ++k) {
        const unsigned long long w = w0 + k * PT;
        unsigned long long win[6];
#pragma unroll
        for (int j = 0; j < 4; ++j) win[j + 1] = r[k][j];
        win[0] = __shfl_up_sync(FULL_MASK, win[4], 1);
        win[5] = __shfl_down_sync(FULL_MASK, win[1], 1);
        if (lane == 0) win[0] = edge[k];
        if (lane == 31) win[5] = edge[k];
        if (w >= Q.n_words) break;
        const long long p0 = (long long)w * 32, p1 = min(p0 + 32, n);
        // the document holding byte p0 (last d with offs[d] <= p0; empty documents
        // skipped): a thread's words ascend, so the search resumes from the last one
        long long hi = dhi;
        while (d < hi) {
            const long long mid = (d + hi + 1) >> 1;
            if (__ldg(&Q.doc_offs[mid]) <= p0) d = mid; else hi = mid - 1;
        }
        while (__ldg(&Q.doc_offs[d + 1]) <= p0) ++d;
        Q.out[w] = word_bits(Q, sasc, p0, p1, win, d);
    }
}

cudaError_t launch_pretok(const PretokParams &Q, cudaStream_t s) {
    if (Q.n_words == 0) return cudaSuccess;
    k_pretok<<<(unsigned int)((Q.n_words + PT * PW - 1) / (PT * PW)), PT, 0, s>>>(Q);
    return cudaGetLastError();
}
