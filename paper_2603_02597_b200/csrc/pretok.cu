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
#include <cuda_runtime.h>

#include "common.cuh"
#include "pretok.cuh"

namespace {

constexpr int PT = 256;      // threads per CTA
constexpr int BACK = 24;     // bytes decoded before a word (>= 4 code points of context)
constexpr int AHEAD = 12;    // bytes decoded after it (2 code points of lookahead)
constexpr int WIN = 32 + BACK + AHEAD;

enum : uint8_t { C_O = 0, C_L = 1, C_N = 2, C_S = 3 };

__device__ __forceinline__ uint8_t cp_class(const PretokParams &Q, uint32_t cp) {
    if (cp >= Q.n_cps) return C_O;
    return (uint8_t)((__ldg(&Q.classes[cp >> 2]) >> (2 * (cp & 3))) & 3u);
}

}  // namespace

__global__ void __launch_bounds__(PT) k_pretok(const __grid_constant__ PretokParams Q) {
    const unsigned long long w = (unsigned long long)blockIdx.x * PT + threadIdx.x;
    if (w >= Q.n_words) return;
    const long long n = (long long)Q.n_bytes;
    const long long p0 = (long long)w * 32, p1 = min(p0 + 32, n);
    // the document holding byte p0 (last d with offs[d] <= p0)
    long long lo = 0, hi = (long long)Q.n_docs - 1;
    while (lo < hi) {
        const long long mid = (lo + hi + 1) >> 1;
        if (__ldg(&Q.doc_offs[mid]) <= p0) lo = mid; else hi = mid - 1;
    }
    long long d = lo;
    uint32_t bits = 0;
    // ---- fast path: one document covers [p0, p1 + 2] and the bytes of
    //      [max(ds, p0 - 4), min(de, p1 + 2)) are ASCII -> code points = bytes
    {
        long long dd = d;
        while (__ldg(&Q.doc_offs[dd + 1]) <= p0) ++dd;
        const long long ds = __ldg(&Q.doc_offs[dd]), de = __ldg(&Q.doc_offs[dd + 1]);
        if (de >= min(n, p1 + 2) || de == n) {
            const long long wlo = max(ds, p0 - 4), whi = min(de, p1 + 2);
            uint8_t wb[40];  // byte p0 - 4 + i, 0 when outside the document
            bool ascii = true;
#pragma unroll
            for (int i = 0; i < 40; ++i) {
                const long long p = p0 - 4 + i;
                const uint8_t b = (p >= wlo && p < whi) ? __ldg(&Q.bytes[p]) : 0u;
                ascii &= b < 0x80u;
                wb[i] = b;
            }
            if (ascii) {
                auto has = [&](int i) { const long long p = p0 - 4 + i; return p >= ds && p < de; };
                auto cls = [&](int i) -> uint8_t { return Q.ascii[wb[i]]; };
                auto tstart = [&](int i) -> bool {
                    if (!has(i - 1)) return true;
                    const uint8_t c = cls(i - 1);
                    return c == C_L || c == C_N || (c == C_S && wb[i - 1] != ' ');
                };
                auto clen = [&](int i) -> int {
                    if (!has(i) || wb[i] != '\'' || !tstart(i)) return 0;
                    const uint8_t a = has(i + 1) ? wb[i + 1] : 0, b = has(i + 2) ? wb[i + 2] : 0;
                    if (a == 's' || a == 'd' || a == 'm' || a == 't') return 2;
                    if ((a == 'l' && b == 'l') || (a == 'v' && b == 'e') || (a == 'r' && b == 'e')) return 3;
                    return 0;
                };
#pragma unroll 4
                for (int k = 0; k < 32; ++k) {
                    const int i = k + 4;
                    if (p0 + k >= p1) break;
                    bool b;
                    if (!has(i - 1)) {
                        b = true;
                    } else if (cls(i) == C_S) {
                        b = cls(i - 1) != C_S || (has(i + 1) && cls(i + 1) != C_S);
                    } else if (cls(i - 1) == C_S) {
                        b = wb[i - 1] != ' ';
                    } else if (clen(i - 1) || clen(i - 2) == 3) {
                        b = false;
                    } else if (clen(i - 2) == 2 || clen(i - 3) == 3) {
                        b = true;
                    } else {
                        b = cls(i) != cls(i - 1);
                    }
                    if (b) bits |= 1u << k;
                }
                Q.out[w] = bits;
                return;
            }
        }
    }
    uint8_t cl[WIN], ch[WIN];
    int16_t at[WIN];
    for (long long pos = p0; pos < p1;) {
        while (__ldg(&Q.doc_offs[d + 1]) <= pos) ++d;  // skip empty documents
        const long long ds = __ldg(&Q.doc_offs[d]), de = __ldg(&Q.doc_offs[d + 1]);
        const long long seg_end = min(p1, de);
        // decode the code points of [q, min(de, seg_end + AHEAD)) of this document
        long long q = max(ds, pos - BACK);
        while (q > ds && q < pos && (__ldg(&Q.bytes[q]) & 0xC0u) == 0x80u) ++q;
        const long long qe = min(de, seg_end + AHEAD);
        int m = 0;
        for (long long i = q; i < qe && m < WIN;) {
            const uint32_t b0 = __ldg(&Q.bytes[i]);
            long long j = i + 1;
            while (j < de && (__ldg(&Q.bytes[j]) & 0xC0u) == 0x80u) ++j;  // continuation bytes join
            uint8_t c = C_O, a = 0;
            if (b0 < 0x80u) {
                c = Q.ascii[b0];
                a = (uint8_t)b0;
            } else {
                const int need = b0 >= 0xF0u ? 3 : b0 >= 0xE0u ? 2 : b0 >= 0xC0u ? 1 : -1;
                if (need > 0 && j - i == need + 1 && b0 < 0xF8u) {
                    uint32_t cp = b0 & (0x3Fu >> need);
                    for (int k = 1; k <= need; ++k) cp = (cp << 6) | (__ldg(&Q.bytes[i + k]) & 0x3Fu);
                    c = cp_class(Q, cp);
                }
            }
            cl[m] = c;
            ch[m] = a;
            at[m] = (int16_t)(i - p0);
            ++m;
            i = j;
        }
        const bool text_start = q == ds;  // cl[0] is the document's first code point
        auto tstart = [&](int j) -> bool {  // token start before code point j (apostrophe test)
            if (j == 0) return text_start;
            return cl[j - 1] == C_L || cl[j - 1] == C_N || (cl[j - 1] == C_S && ch[j - 1] != ' ');
        };
        auto clen = [&](int j) -> int {  // contraction starting at code point j: its length, else 0
            if (j < 0 || j >= m || ch[j] != '\'' || !tstart(j)) return 0;
            const uint8_t a = j + 1 < m ? ch[j + 1] : 0, b = j + 2 < m ? ch[j + 2] : 0;
            if (a == 's' || a == 'd' || a == 'm' || a == 't') return 2;
            if ((a == 'l' && b == 'l') || (a == 'v' && b == 'e') || (a == 'r' && b == 'e')) return 3;
            return 0;
        };
        for (int k = 0; k < m; ++k) {
            const long long p = p0 + at[k];
            if (p < pos) continue;
            if (p >= seg_end) break;
            bool b;
            if (k == 0) {
                b = text_start;  // (a word never starts BACK bytes into a document's interior)
            } else if (cl[k] == C_S) {
                b = cl[k - 1] != C_S || (k + 1 < m && cl[k + 1] != C_S);
            } else if (cl[k - 1] == C_S) {
                b = ch[k - 1] != ' ';
            } else if (clen(k - 1)) {
                b = false;
            } else if (clen(k - 2) == 3) {
                b = false;
            } else if (clen(k - 2) == 2 || clen(k - 3) == 3) {
                b = true;
            } else {
                b = cl[k] != cl[k - 1];
            }
            if (b) bits |= 1u << at[k];
        }
        pos = seg_end;
    }
    Q.out[w] = bits;
}

cudaError_t launch_pretok(const PretokParams &Q, cudaStream_t s) {
    if (Q.n_words == 0) return cudaSuccess;
    k_pretok<<<(unsigned int)((Q.n_words + PT - 1) / PT), PT, 0, s>>>(Q);
    return cudaGetLastError();
}
