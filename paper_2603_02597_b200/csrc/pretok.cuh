// pretok.cuh -- parameters of the GPT-2 regex pre-tokenization pass (pretok.cu).
#pragma once
#include <cstdint>

struct PretokParams {
    const uint8_t *bytes;
    unsigned long long n_bytes;
    const long long *doc_offs;     // [n_docs + 1]
    unsigned long long n_docs;
    const uint8_t *classes;        // 2-bit code point classes (O, L, N, \s), 4 per byte
    uint32_t n_cps;                // code points covered by `classes`
    uint8_t ascii[128];            // classes of the ASCII code points
    uint32_t paths;                // fast paths enabled: 1 SWAR, 2 ASCII masks, 4 Unicode masks (else scalar)
    uint32_t ascii_std;            // ascii[] is L = [A-Za-z], N = [0-9], \s = [\t-\r ] (bit-parallel path)
    uint32_t *out;                 // [n_words] token-start bits
    unsigned long long n_words;
};

#ifdef __CUDACC__
cudaError_t launch_pretok(const PretokParams &Q, cudaStream_t s);
#endif
