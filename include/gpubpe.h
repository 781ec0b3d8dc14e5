/*
 * gpubpe.h -- C ABI of the B200 GPT-2 byte-level BPE encoder.
 *
 * This is the drop-in boundary for the reference's encode path
 * (/root/reference/pkg, package `lanebpe`).  The reference is pure Python, so
 * its "FFI" is its Python call surface; each entry point below names the
 * reference interface it replaces.  A maintainer binds it with ctypes (see
 * INTEGRATION.md); paper_2603_02597_b200/_native.py is exactly that binding.
 *
 * Conventions: plain pointers and sizes, no torch types.  Pointers prefixed
 * d_ are device (HBM) pointers on the context's device; h_ are host pointers.
 * Every function returns 0 on success or a GPUBPE_E* code; the message of the
 * last failure is available from gpubpe_last_error().  A context is not
 * thread-safe: callers serialise use of one context (the Python layer holds a
 * lock), or create one context per thread.
 */
#ifndef GPUBPE_H
#define GPUBPE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GPUBPE_OK 0
#define GPUBPE_EINVAL 1     /* bad argument (maps to ValueError / InvalidBudget) */
#define GPUBPE_ECUDA 2      /* CUDA runtime / launch failure (DeviceError) */
#define GPUBPE_ENOMEM 3     /* device or host allocation failed (DeviceError) */
#define GPUBPE_ETABLE 4     /* merge table rejected: duplicate pair / reserved key */
#define GPUBPE_ERANGE 5     /* output capacity too small (the needed size is reported) */

#define GPUBPE_API_VERSION 1

typedef struct gpubpe_ctx gpubpe_ctx;

/* Counters of the last encode (lanebpe PassCounters, engines.py:77-97, plus
 * device-side evidence).  passes == n_bytes - n_ids always
 * (test_acceptance.py:363-376). */
typedef struct gpubpe_stats {
    uint64_t n_bytes;          /* base tokens in (one per byte) */
    uint64_t n_ids;            /* ids out */
    uint64_t passes;           /* merges applied = n_bytes - n_ids */
    uint64_t n_segments;       /* junction segments (incl. chunk / doc cuts) */
    uint64_t memo_hits;        /* segments resolved by one memo probe */
    uint64_t short_merges;     /* memo-miss segments (<= 32 B) merged by the sequential warp engine */
    uint64_t medium_segments;  /* segments merged by the CTA engine in smem */
    uint64_t giant_segments;   /* segments merged by the giant (multi-window) engine */
    uint64_t giant_bytes;      /* bytes inside giant segments */
    uint64_t engine_passes;    /* warp-engine steps + multi-merge passes of the medium/giant engines */
    uint64_t tiles;            /* encode tiles launched */
    uint64_t overflow;         /* 1 if the giant arena overflowed (call re-run) */
    uint64_t well_formed;      /* 1 if the table admits exact multi-merge passes */
    uint64_t allocations;      /* device / pinned buffers allocated by the last call
                                  (0 in steady state: workspaces are grow-only;
                                  PassCounters.buffer_allocations) */
} gpubpe_stats;

/* Context flags */
#define GPUBPE_F_NO_MEMO 1u      /* disable the vocab-string memo (evidence runs) */
#define GPUBPE_F_STRICT 2u       /* force one-merge-per-pass even if well-formed */
#define GPUBPE_F_HOST_TABLES 4u  /* build the junction bitmap with the host loops (parity checks) */

/* Encode modes (gpubpe_set_mode) */
#define GPUBPE_MODE_DEFAULT 0u     /* the reference's semantics: no pre-tokenization */
#define GPUBPE_MODE_GPT2_REGEX 1u  /* tiktoken's GPT-2 regex pre-tokens are cuts too (optional) */

/*
 * Build a device context (replaces Tokenizer.__init__ / Tokenizer.from_files,
 * chunker.py:74-93, and build_table, merge_table.py:246-278, as the place the
 * tables are materialised).
 *   base_ids[256]        byte -> token id (byte_codec.py:97-111)
 *   left/right/rank/new  n_rules merge rules (merge_table.py:80-116)
 *   vocab_ids/bytes/offs n_vocab tokens with their byte strings (symbols
 *                        containing non-byte characters omitted); used for the
 *                        vocab-string memo, which is verified on the device at
 *                        creation time (only strings whose BPE is themselves)
 *   flags                GPUBPE_F_*
 * Errors: GPUBPE_ETABLE for a duplicate (left,right) pair (DuplicatePair).
 */
int gpubpe_ctx_create(int device, const uint32_t *base_ids, const uint32_t *left,
                      const uint32_t *right, const uint32_t *rank, const uint32_t *new_tok,
                      uint64_t n_rules, const uint32_t *vocab_ids, const uint8_t *vocab_bytes,
                      const uint64_t *vocab_offs, uint64_t n_vocab, uint32_t flags,
                      gpubpe_ctx **out);

/*
 * Encode a packed batch (replaces tokenize_batch, chunker.py:110-187, with
 * the sequential engine's output, engines.py:269-335).
 *   d_bytes[n_bytes]          all documents back to back (uint8)
 *   d_doc_offs[n_docs+1]      int64 CSR offsets, d_doc_offs[0] == 0,
 *                             d_doc_offs[n_docs] == n_bytes
 *   max_seq_len, chunk_budget BlockConfig (engines.py:40-65): a document longer
 *                             than max_seq_len is cut at multiples of
 *                             chunk_budget (chunker.py:42-53,139-144)
 *   d_out_ids                 capacity n_bytes uint32 ids
 *   d_out_offs[n_docs+1]      int64 CSR offsets of the ids
 *   stream                    cudaStream_t (NULL = legacy default stream)
 * Asynchronous: returns once the kernel is enqueued, except when the input
 * is large enough that the giant-segment arena might overflow, in which case
 * it synchronises the stream and re-runs with a larger arena.
 */
int gpubpe_encode(gpubpe_ctx *ctx, const uint8_t *d_bytes, uint64_t n_bytes,
                  const int64_t *d_doc_offs, uint64_t n_docs, uint64_t max_seq_len,
                  uint64_t chunk_budget, uint32_t *d_out_ids, int64_t *d_out_offs,
                  void *stream);

/*
 * Encode from and to HOST memory -- the reference's own call shape (bytes in,
 * ids out; tokenize_batch, chunker.py:110-187, for a packed batch).  Stages
 * the batch into context-owned pinned memory (several threads), copies it to
 * the device in one H2D copy and launches the same encode as gpubpe_encode
 * behind it (128 KiB .. 16 MiB: on the caller's stream while the copy is in
 * flight, the tiles waiting for an arrival word); the kernel writes the ids
 * and offsets straight into pinned, device-mapped host memory (the caller's
 * h_out_ids when it comes from gpubpe_host_alloc) and its last CTA publishes
 * the id count and counters there too, so the call returns as soon as they
 * are visible (no device-to-host copy).  Batches above 64 MiB stream through
 * a two-slot H2D / encode / D2H pipeline.  Synchronous for the caller.
 *   h_out_ids      capacity >= n_bytes (ids <= bytes)
 *   h_out_offs     n_docs+1 int64 CSR offsets of the ids
 *   n_ids_out      ids written
 *   kernel_ms      nullable: device time of the encode (CUDA events; the
 *                  host's enqueue-to-results time when the events are not
 *                  complete yet)
 */
int gpubpe_encode_host(gpubpe_ctx *ctx, const uint8_t *h_bytes, uint64_t n_bytes,
                       const int64_t *h_doc_offs, uint64_t n_docs, uint64_t max_seq_len,
                       uint64_t chunk_budget, uint32_t *h_out_ids, int64_t *h_out_offs,
                       uint64_t *n_ids_out, float *kernel_ms, void *stream);

/* Pinned, device-mapped host memory for results: when gpubpe_encode_host's
 * h_out_ids points into such a buffer the kernel writes the ids there
 * directly (no copy-out).  Free with gpubpe_host_free. */
int gpubpe_host_alloc(int device, uint64_t bytes, void **out);
void gpubpe_host_free(void *p);

/* Synchronise `stream` and read the counters of the last encode on it
 * (BatchResult.counters, chunker.py:56-64). */
int gpubpe_query(gpubpe_ctx *ctx, void *stream, gpubpe_stats *out);

/*
 * Device decode, ids -> bytes (replaces decode_tokens, byte_codec.py:121-146,
 * and Tokenizer.decode, chunker.py:100-101).
 * gpubpe_set_vocab: the byte string of every decodable id (n strings; ids
 *   absent here, or with symbols containing non-byte characters, are unknown).
 *   Empty strings (an empty symbol decodes to no bytes) and strings of any
 *   length below 2 GiB are decodable.
 * gpubpe_decode: d_ids[n_ids] as n_seqs sequences (d_id_offs[n_seqs+1] CSR;
 *   n_seqs == 0: one sequence, no offsets) -> their byte strings back to back
 *   in d_out (capacity out_cap) with d_out_offs[n_seqs+1].  Synchronises.
 *   d_out must be 16-byte aligned (the kernels store 16-byte vectors) and
 *   d_ids 4-byte aligned; a misaligned pointer is GPUBPE_EINVAL, never a
 *   fault.
 *   Unknown id: GPUBPE_EINVAL, *bad_index = its index (UnknownTokenId).
 *   Capacity too small: GPUBPE_ERANGE, *n_bytes_out = the bytes needed.
 */
int gpubpe_set_vocab(gpubpe_ctx *ctx, const uint32_t *ids, const uint8_t *bytes, const uint64_t *offs,
                     uint64_t n);
int gpubpe_decode(gpubpe_ctx *ctx, const uint32_t *d_ids, uint64_t n_ids, const int64_t *d_id_offs,
                  uint64_t n_seqs, uint8_t *d_out, uint64_t out_cap, int64_t *d_out_offs,
                  uint64_t *n_bytes_out, uint64_t *bad_index, void *stream);

/*
 * Optional GPT-2 regex pre-tokenization (not the reference's
 * semantics, which has none -- SPEC.md:93,95 -- so never the default).
 * gpubpe_set_pretok: 2-bit classes (0 other, 1 \p{L}, 2 \p{N}, 3 \s) of
 *   code points 0..n_cps-1, four per byte.
 * gpubpe_set_mode: GPUBPE_MODE_DEFAULT or GPUBPE_MODE_GPT2_REGEX for the
 *   following encodes of this context (gpubpe_encode / gpubpe_encode_host):
 *   the tokens of tiktoken's GPT-2 pattern become additional cut points, so
 *   the ids are tiktoken's GPT-2 encode_ordinary ids for valid UTF-8 text.
 */
int gpubpe_set_pretok(gpubpe_ctx *ctx, const uint8_t *classes, uint64_t n_cps);
int gpubpe_set_mode(gpubpe_ctx *ctx, uint32_t mode);

/* The junction bitmap of the context (65,536 bits as uint32[2048]; bit
 * (x << 8 | y) set iff some reachable rule joins a token ending in byte x to
 * one starting with byte y).  A byte pair outside it is a cut no merge of
 * the reference can span, so a document may be split there across GPUs
 * (multigpu.py). */
int gpubpe_junction_bits(gpubpe_ctx *ctx, uint32_t *h_out);

/* Token-level merges (replaces sequential_bpe, engines.py:269-335, and the
 * output of run_block_engine, engines.py:338-403): for each sequence s of
 * device tokens d_tokens[h_offs[s] .. h_offs[s+1]) the greedy lowest-rank /
 * leftmost BPE fixpoint is written to d_out at the same offset, its length in
 * h_counts[s] (host).  Every token must be an id the merge table covers
 * (< the context's id bound; GPUBPE_EINVAL names the sequence otherwise) and
 * ids must be below 2^24.  Synchronous. */
int gpubpe_merge_tokens(gpubpe_ctx *ctx, const uint32_t *d_tokens, const uint64_t *h_offs, uint64_t n_seqs,
                        uint32_t *d_out, uint64_t *h_counts, void *stream);

/* gpubpe_merge_tokens plus the reference's two debugging hooks of the engine:
 *   d_trace    nullable, device, one uint64 per input token (same offsets as
 *              d_tokens): merge k of sequence s stores (pass << 34) | (merged
 *              at position 0 << 33) | (its right token was the last << 32) |
 *              rank at d_trace[h_offs[s] + k], in pass order and by position
 *              inside a pass -- the first/last bits give sequential_bpe's
 *              lookup count (a merge probes each neighbour it has); the
 *              `trace` argument of sequential_bpe /
 *              run_block_engine (engines.py:270,317-319,395-396) is the ranks
 *              in this order when passes merge one pair (tables that are not
 *              well-formed), and sorted by rank otherwise;
 *   fault_seq  -1, or the sequence whose run applies inject_compaction_fault
 *              (engines.py:252-266,378-388): the first pass that can be
 *              corrupted merges its winning pair one slot off (p+1, else p-1)
 *              with the winner's new token.
 * Id n_ids of the context (one past the largest id of its tables) is an inert
 * token no rule mentions: callers map ids outside the table to it. */
int gpubpe_merge_tokens_ex(gpubpe_ctx *ctx, const uint32_t *d_tokens, const uint64_t *h_offs, uint64_t n_seqs,
                           uint32_t *d_out, uint64_t *h_counts, uint64_t *d_trace, int64_t fault_seq,
                           void *stream);

/* One evaluation pass of the reference's lane engine (eval_pairs,
 * engines.py:133-168) on the device: probe every adjacent pair of
 * d_tokens[0..n) and reduce to the lowest rank, leftmost on ties.
 * h_result[0] = position (UINT64_MAX when no pair is in the table),
 * h_result[1] = rank, h_result[2] = new token id.  Synchronous. */
int gpubpe_eval_pairs(gpubpe_ctx *ctx, const uint32_t *d_tokens, uint64_t n, uint64_t *h_result, void *stream);

/* One merge applied by compaction (engines.py:171-217): d_out[0..n-1) =
 * d_tokens with slots best_pos, best_pos+1 replaced by new_token.
 * method 0 = compact_double_buffer (direct index map), 1 = compact_scan
 * (removal flags + exclusive prefix sum + scatter).  GPUBPE_EINVAL when
 * best_pos is not a pair position (OutOfRange).  Asynchronous, on the
 * current device. */
int gpubpe_compact(const uint32_t *d_tokens, uint64_t n, uint64_t best_pos, uint32_t new_token, uint32_t *d_out,
                   int method, void *stream);

/* PackedPairTable.lookup_keys_into (merge_table.py:170-230) on the device:
 * packed keys (left << 32) | right -> d_hit[i] (0/1) and d_vals[i] =
 * (new << 32) | rank where hit; the empty-slot key UINT64_MAX is a miss.
 * Asynchronous. */
int gpubpe_lookup_keys(gpubpe_ctx *ctx, const uint64_t *d_keys, uint64_t m, uint8_t *d_hit, uint64_t *d_vals,
                       void *stream);

/* Device-side merges parsing; replaces the line loop
 * of parse_merges (merge_table.py:88-116) with its vocabulary lookups
 * (byte_codec.py:80-88).  The vocabulary is given as UTF-8 symbols in CSR form
 * (sym_bytes, sym_offs[n_syms+1]) with their ids; line i of the merges text
 * is text[line_start[i], line_end[i]) (line breaks and the optional "#"
 * header removed by the caller).  For every line: out_status[i] = 0 and the
 * ids of a, b and a+b in out_left/out_right/out_new, or 1 (not exactly two
 * nonempty space-separated symbols: MalformedLine) or 2 (a symbol missing
 * from the vocabulary: UnknownSymbol).  Ranks are the line indices. */
int gpubpe_parse_merges(int device, const uint8_t *sym_bytes, const uint64_t *sym_offs,
                        const uint32_t *sym_ids, uint64_t n_syms, const uint8_t *text, uint64_t text_len,
                        const uint64_t *line_start, const uint64_t *line_end, uint64_t n_lines,
                        uint32_t *out_left, uint32_t *out_right, uint32_t *out_new, uint8_t *out_status);

/* Number of kernels one gpubpe_encode enqueues (launch accounting): 1, the
 * fused persistent k_encode. */
int gpubpe_launches_per_encode(void);

/* gpubpe_encode_host for a batch given as n_docs separate host buffers
 * (h_ptrs[d], h_lens[d]): the documents are gathered (in parallel) straight
 * into the pinned staging buffer -- one host copy instead of a join plus a
 * staging copy.  Same outputs and errors as gpubpe_encode_host. */
int gpubpe_encode_host_gather(gpubpe_ctx *ctx, const uint64_t *h_ptrs, const uint64_t *h_lens, uint64_t n_docs,
                              uint64_t max_seq_len, uint64_t chunk_budget, uint32_t *h_out_ids,
                              int64_t *h_out_offs, uint64_t *n_ids_out, float *kernel_ms, void *stream);

/* Device-side probe of the packed pair table: for i < n, (d_left[i],
 * d_right[i]) -> d_new[i], d_rank[i] (0xFFFFFFFF rank on miss).  Replaces
 * PackedPairTable.lookup_pairs (merge_table.py:232-243); used by the table
 * conformance tests. */
int gpubpe_lookup_pairs(gpubpe_ctx *ctx, const uint32_t *d_left, const uint32_t *d_right,
                        uint64_t n, uint32_t *d_new, uint32_t *d_rank, void *stream);

/* Kernel timing of subsequent encodes: when on, CUDA events are recorded on
 * the encode stream around the encode kernel (k_encode).  gpubpe_kernel_ms
 * synchronises on the last encode and writes its kernel duration in ms to
 * ms[0] (n >= 1). */
int gpubpe_set_profiling(gpubpe_ctx *ctx, int on);
int gpubpe_kernel_ms(gpubpe_ctx *ctx, float *ms, int n);

const char *gpubpe_last_error(gpubpe_ctx *ctx);
void gpubpe_ctx_destroy(gpubpe_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* GPUBPE_H */
