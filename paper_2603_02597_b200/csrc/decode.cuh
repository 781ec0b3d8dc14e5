// decode.cuh -- parameters of the device decode (ids -> bytes), decode.cu.
#pragma once
#include <cstdint>

constexpr uint32_t LEN_EXT = 255;

struct DecodeState {
    unsigned long long tile_ctr;
    unsigned long long need;     // output bytes needed when out_cap was too small
    unsigned long long n_bytes;  // bytes written
    unsigned long long bad;      // smallest index of an unknown id, ~0 if none
};

struct DecodeParams {
    // Lengths: 1..254 in place; LEN_EXT (255) marks an id whose length is 0 (an
    // empty symbol) or >= 255 -- its exact length is in vlong (and vrec's .z).
    const uint32_t *vinfo;  // per id: blob offset << 8 | min(length, LEN_EXT), INF if not decodable
    const uint8_t *blob;
    const uint4 *vrec;      // per id: 16-B record, byte 0 = length (0 for empty symbols); length
                            // <= 15: the string in bytes 1..15, else .y = its blob chunk (offset / 16)
                            // and byte 0 = min(length, LEN_EXT), .z = the length; zero if unknown;
                            // n_vocab + 1 records (the last one zero)
    const uint8_t *vlen;    // per id: length (LEN_EXT: see vlong), 0 if not decodable
    const uint32_t *vlong;  // per id: exact length (read only behind LEN_EXT)
    uint32_t ext;           // the vocabulary has LEN_EXT lengths (kernels instantiated for them)
    uint32_t n_vocab;       // ids >= n_vocab are unknown
    const uint32_t *ids;
    unsigned long long n_ids;
    const long long *id_offs;  // [n_seqs + 1] CSR of id sequences (nullable when n_seqs == 0)
    unsigned long long n_seqs;
    uint8_t *out;
    unsigned long long out_cap;
    long long *out_offs;       // [n_seqs + 1] byte offsets
    DecodeState *st;
    unsigned long long *status;  // [n_tiles] look-back words (single-pass mode)
    const unsigned long long *tile_base;  // [n_tiles] output offset of each tile (two-pass mode), or null
    uint32_t *row_bytes;       // [n_tiles * 32] bytes of each 128-id row (two-pass mode), or null
    unsigned long long n_tiles;
    unsigned int epoch;
    int aligned;               // ids pointer is 16-B aligned
};

#ifdef __CUDACC__
size_t decode_smem_bytes();
int decode_tile_ids();
cudaError_t setup_decode();
cudaError_t decode_occupancy(int *blocks);
cudaError_t launch_decode(const DecodeParams &P, int grid, cudaStream_t s);
cudaError_t decode_rows_occupancy(int *blocks);
cudaError_t launch_decode_rows(const DecodeParams &P, int grid, cudaStream_t s);
cudaError_t launch_decode_offsets(const DecodeParams &P, unsigned long long *tile_bytes,
                                  unsigned long long *tile_base, cudaStream_t s);
#endif
