// build.cu -- device-side table construction.
//
// Two one-time jobs of the reference's cold start move to the GPU:
//   * merges.txt parsing (merge_table.py:88-116 parse_merges): every line is
//     "a b"; a, b and a+b are looked up in the vocabulary (byte_codec.py:80-88).
//     The vocabulary's UTF-8 symbols go into an open-addressing hash on the
//     device, then one thread per line splits it and looks its three symbols
//     up; a per-line status (ok / malformed / unknown symbol) lets the host
//     raise exactly the reference's first error;
//   * the junction bitmap J of the encode context (ctx.cu): the first/last
//     byte sets F(t), B(t) of every token are the least fixpoint of
//     F(new) |= F(left), B(new) |= B(right) from the base bytes (one kernel
//     sweep over the rules per round until nothing changes), then
//     J[x] |= F(right) for every x in B(left) of every rule.
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "../../include/gpubpe.h"
#include "common.cuh"

namespace {

constexpr unsigned long long SLOT_EMPTY = ~0ull;

__host__ __device__ __forceinline__ uint64_t sym_hash_step(uint64_t h, uint8_t b) {
    return (h ^ b) * 0x100000001B3ull;  // FNV-1a, 64-bit
}
constexpr uint64_t SYM_HASH_INIT = 0xCBF29CE484222325ull;

struct SymTable {
    const uint8_t *bytes;    // UTF-8 of every symbol, back to back
    const uint64_t *offs;    // [n + 1]
    const uint32_t *ids;     // [n]
    unsigned long long *slots;  // (hash >> 32) << 32 | symbol index; SLOT_EMPTY when free
    uint32_t mask;
};

__global__ void k_sym_insert(SymTable S, uint64_t n) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t h = SYM_HASH_INIT;
    for (uint64_t p = S.offs[i]; p < S.offs[i + 1]; ++p) h = sym_hash_step(h, S.bytes[p]);
    const unsigned long long v = ((h >> 32) << 32) | (uint32_t)i;
    uint32_t s = (uint32_t)h & S.mask;
    while (atomicCAS(&S.slots[s], SLOT_EMPTY, v) != SLOT_EMPTY) s = (s + 1) & S.mask;
}

// Id of the symbol whose UTF-8 is text[a0, a1) ++ text[b0, b1), or INF.
__device__ uint32_t sym_lookup(const SymTable &S, const uint8_t *text, uint64_t a0, uint64_t a1, uint64_t b0,
                               uint64_t b1) {
    uint64_t h = SYM_HASH_INIT;
    for (uint64_t p = a0; p < a1; ++p) h = sym_hash_step(h, text[p]);
    for (uint64_t p = b0; p < b1; ++p) h = sym_hash_step(h, text[p]);
    const uint64_t len = (a1 - a0) + (b1 - b0);
    for (uint32_t s = (uint32_t)h & S.mask;; s = (s + 1) & S.mask) {
        const unsigned long long v = S.slots[s];
        if (v == SLOT_EMPTY) return GPUBPE_INF;
        if ((v >> 32) != (h >> 32)) continue;
        const uint32_t k = (uint32_t)v;
        const uint64_t o = S.offs[k];
        if (S.offs[k + 1] - o != len) continue;
        bool eq = true;
        for (uint64_t p = 0; p < len && eq; ++p) {
            const uint64_t q = p < a1 - a0 ? a0 + p : b0 + (p - (a1 - a0));
            eq = S.bytes[o + p] == text[q];
        }
        if (eq) return S.ids[k];
    }
}

// One thread per line [ls, le): status 0 ok, 1 malformed (not exactly two
// nonempty space-separated symbols), 2 a symbol missing from the vocabulary.
__global__ void k_parse_lines(SymTable S, const uint8_t *text, const uint64_t *ls, const uint64_t *le, uint64_t n,
                              uint32_t *left, uint32_t *right, uint32_t *nw, uint8_t *status) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t s = ls[i], e = le[i];
    uint64_t sp = 0;
    uint32_t nsp = 0;
    for (uint64_t p = s; p < e; ++p)
        if (text[p] == ' ') {
            ++nsp;
            sp = p;
        }
    if (nsp != 1 || sp == s || sp + 1 == e) {
        status[i] = 1;
        return;
    }
    const uint32_t a = sym_lookup(S, text, s, sp, sp, sp);
    const uint32_t b = sym_lookup(S, text, sp + 1, e, e, e);
    const uint32_t ab = sym_lookup(S, text, s, sp, sp + 1, e);
    if (a == GPUBPE_INF || b == GPUBPE_INF || ab == GPUBPE_INF) {
        status[i] = 2;
        return;
    }
    left[i] = a;
    right[i] = b;
    nw[i] = ab;
    status[i] = 0;
}

// One round of F(new) |= F(left), B(new) |= B(right) over every rule.
__global__ void k_fb_round(const uint32_t *L, const uint32_t *R, const uint32_t *NW, uint64_t n,
                           unsigned long long *F, unsigned long long *B, int *changed) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t t = NW[i], l = L[i], r = R[i];
    bool ch = false;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        const unsigned long long f = F[l * 4 + w], b = B[r * 4 + w];
        if (f & ~F[t * 4 + w]) {
            atomicOr(&F[t * 4 + w], f);
            ch = true;
        }
        if (b & ~B[t * 4 + w]) {
            atomicOr(&B[t * 4 + w], b);
            ch = true;
        }
    }
    if (ch) *changed = 1;
}

// J[x] |= F(right) for every last byte x of left, every rule (one thread per
// rule and 64-bit word of B(left)).
__global__ void k_junction(const uint32_t *L, const uint32_t *R, uint64_t n, const unsigned long long *F,
                           const unsigned long long *B, unsigned long long *J) {
    const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t i = g >> 2;
    const int wx = (int)(g & 3);
    if (i >= n) return;
    const uint64_t l = L[i], r = R[i];
    unsigned long long bx = B[l * 4 + wx];
    const unsigned long long f0 = F[r * 4], f1 = F[r * 4 + 1], f2 = F[r * 4 + 2], f3 = F[r * 4 + 3];
    while (bx) {
        const int x = wx * 64 + __ffsll((long long)bx) - 1;
        bx &= bx - 1;
        if (f0) atomicOr(&J[x * 4], f0);
        if (f1) atomicOr(&J[x * 4 + 1], f1);
        if (f2) atomicOr(&J[x * 4 + 2], f2);
        if (f3) atomicOr(&J[x * 4 + 3], f3);
    }
}

template <typename T>
struct DBuf {  // device buffer freed on scope exit
    T *p = nullptr;
    cudaError_t alloc(size_t n) { return cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)); }
    ~DBuf() {
        if (p) cudaFree(p);
    }
};

#define BK(call)                                  \
    do {                                          \
        cudaError_t e_ = (call);                  \
        if (e_ != cudaSuccess) return e_;         \
    } while (0)

}  // namespace

// Junction bitmap on the device (ctx.cu calls this with the interned rules).
// jbits: 2048 words, bit (x << 8 | y).
cudaError_t build_junction_device(const uint32_t *h_base, const uint32_t *h_L, const uint32_t *h_R,
                                  const uint32_t *h_NW, uint64_t n_rules, uint64_t n_ids, uint32_t *h_jbits,
                                  int *h_rounds) {
    DBuf<uint32_t> L, R, NW;
    DBuf<unsigned long long> F, B, J;
    DBuf<int> changed;
    BK(L.alloc(n_rules));
    BK(R.alloc(n_rules));
    BK(NW.alloc(n_rules));
    BK(F.alloc(n_ids * 4));
    BK(B.alloc(n_ids * 4));
    BK(J.alloc(1024));
    BK(changed.alloc(1));
    if (n_rules) {
        BK(cudaMemcpy(L.p, h_L, n_rules * 4, cudaMemcpyHostToDevice));
        BK(cudaMemcpy(R.p, h_R, n_rules * 4, cudaMemcpyHostToDevice));
        BK(cudaMemcpy(NW.p, h_NW, n_rules * 4, cudaMemcpyHostToDevice));
    }
    std::vector<unsigned long long> f0(n_ids * 4, 0);
    for (int b = 0; b < 256; ++b) f0[(uint64_t)h_base[b] * 4 + (b >> 6)] |= 1ull << (b & 63);
    BK(cudaMemcpy(F.p, f0.data(), f0.size() * 8, cudaMemcpyHostToDevice));
    BK(cudaMemcpy(B.p, f0.data(), f0.size() * 8, cudaMemcpyHostToDevice));
    BK(cudaMemset(J.p, 0, 1024 * 8));
    const unsigned int grid = (unsigned int)((n_rules + 255) / 256);
    int rounds = 0;
    for (int ch = 1; ch && n_rules;) {
        BK(cudaMemset(changed.p, 0, sizeof(int)));
        k_fb_round<<<grid, 256>>>(L.p, R.p, NW.p, n_rules, F.p, B.p, changed.p);
        BK(cudaGetLastError());
        BK(cudaMemcpy(&ch, changed.p, sizeof(int), cudaMemcpyDeviceToHost));
        ++rounds;
    }
    if (n_rules) {
        k_junction<<<(unsigned int)((4 * n_rules + 255) / 256), 256>>>(L.p, R.p, n_rules, F.p, B.p, J.p);
        BK(cudaGetLastError());
    }
    std::vector<unsigned long long> hj(1024);
    BK(cudaMemcpy(hj.data(), J.p, 1024 * 8, cudaMemcpyDeviceToHost));
    for (int k = 0; k < 2048; ++k) h_jbits[k] = (uint32_t)(hj[k >> 1] >> (32 * (k & 1)));
    if (h_rounds) *h_rounds = rounds;
    return cudaSuccess;
}

extern "C" __attribute__((visibility("default"))) int gpubpe_parse_merges(
    int device, const uint8_t *sym_bytes, const uint64_t *sym_offs, const uint32_t *sym_ids, uint64_t n_syms,
    const uint8_t *text, uint64_t text_len, const uint64_t *line_start, const uint64_t *line_end,
    uint64_t n_lines, uint32_t *out_left, uint32_t *out_right, uint32_t *out_new, uint8_t *out_status) {
    if ((n_syms && (!sym_bytes || !sym_offs || !sym_ids)) || (n_lines && (!text || !line_start || !line_end)) ||
        (n_lines && (!out_left || !out_right || !out_new || !out_status)))
        return GPUBPE_EINVAL;
    if (n_syms >= (1ull << 32)) return GPUBPE_EINVAL;
    if (cudaSetDevice(device) != cudaSuccess) return GPUBPE_ECUDA;
    if (n_lines == 0) return GPUBPE_OK;
    auto run = [&]() -> cudaError_t {
        uint64_t cap = 2;
        while (cap < 2 * std::max<uint64_t>(n_syms, 1)) cap <<= 1;
        const uint64_t nb = sym_offs[n_syms];
        DBuf<uint8_t> db, dt, dst;
        DBuf<uint64_t> doffs, dls, dle;
        DBuf<uint32_t> dids, dl, dr, dn;
        DBuf<unsigned long long> dslots;
        BK(db.alloc(nb));
        BK(doffs.alloc(n_syms + 1));
        BK(dids.alloc(n_syms));
        BK(dslots.alloc(cap));
        BK(dt.alloc(text_len));
        BK(dls.alloc(n_lines));
        BK(dle.alloc(n_lines));
        BK(dl.alloc(n_lines));
        BK(dr.alloc(n_lines));
        BK(dn.alloc(n_lines));
        BK(dst.alloc(n_lines));
        if (nb) BK(cudaMemcpy(db.p, sym_bytes, nb, cudaMemcpyHostToDevice));
        BK(cudaMemcpy(doffs.p, sym_offs, (n_syms + 1) * 8, cudaMemcpyHostToDevice));
        if (n_syms) BK(cudaMemcpy(dids.p, sym_ids, n_syms * 4, cudaMemcpyHostToDevice));
        if (text_len) BK(cudaMemcpy(dt.p, text, text_len, cudaMemcpyHostToDevice));
        BK(cudaMemcpy(dls.p, line_start, n_lines * 8, cudaMemcpyHostToDevice));
        BK(cudaMemcpy(dle.p, line_end, n_lines * 8, cudaMemcpyHostToDevice));
        BK(cudaMemset(dslots.p, 0xFF, cap * 8));
        SymTable S{db.p, doffs.p, dids.p, dslots.p, (uint32_t)(cap - 1)};
        if (n_syms) {
            k_sym_insert<<<(unsigned int)((n_syms + 255) / 256), 256>>>(S, n_syms);
            BK(cudaGetLastError());
        }
        k_parse_lines<<<(unsigned int)((n_lines + 255) / 256), 256>>>(S, dt.p, dls.p, dle.p, n_lines, dl.p, dr.p,
                                                                       dn.p, dst.p);
        BK(cudaGetLastError());
        BK(cudaMemcpy(out_left, dl.p, n_lines * 4, cudaMemcpyDeviceToHost));
        BK(cudaMemcpy(out_right, dr.p, n_lines * 4, cudaMemcpyDeviceToHost));
        BK(cudaMemcpy(out_new, dn.p, n_lines * 4, cudaMemcpyDeviceToHost));
        BK(cudaMemcpy(out_status, dst.p, n_lines, cudaMemcpyDeviceToHost));
        return cudaSuccess;
    };
    const cudaError_t e = run();
    if (e != cudaSuccess) return e == cudaErrorMemoryAllocation ? GPUBPE_ENOMEM : GPUBPE_ECUDA;
    return GPUBPE_OK;
}
