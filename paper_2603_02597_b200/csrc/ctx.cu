// ctx.cu -- host side of the C ABI (include/gpubpe.h): table construction,
// workspace management, launch and counters.
//
// Construction restates what the reference derives from its inputs
// (byte_codec.py:97-111 base ids, merge_table.py:246-278 the pair table with
// DuplicatePair detection) and adds the device-only structures described in
// common.cuh (rl/rr, junction bitmap, well-formedness, verified memo).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/gpubpe.h"
#include "kernels.cuh"
#include "decode.cuh"
#include "pretok.cuh"
#include "tokens.cuh"

size_t tile_smem_bytes();
cudaError_t launch_encode(const EncodeParams &P, int grid, cudaStream_t s, cudaEvent_t *ev,
                          const cudaAccessPolicyWindow *win, bool coop);
cudaError_t setup_kernels();
cudaError_t tile_occupancy(int *blocks);
cudaError_t build_junction_device(const uint32_t *h_base, const uint32_t *h_L, const uint32_t *h_R,
                                  const uint32_t *h_NW, uint64_t n_rules, uint64_t n_ids, uint32_t *h_jbits,
                                  int *h_rounds);
cudaError_t launch_lookup(const DevTables &T, const uint32_t *l, const uint32_t *r,
                          unsigned long long n, uint32_t *nw, uint32_t *rank, cudaStream_t s);

namespace {

struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
};

}  // namespace

struct gpubpe_ctx {
    int device = 0;
    int num_sms = 0;
    int tile_blocks_per_sm = 1;
    uint32_t flags = 0;
    DevTables T{};
    // all device tables live in one allocation, pinned in L2 by an access
    // policy window on every encode launch
    uint8_t *tables = nullptr;
    size_t tables_bytes = 0, tables_used = 0;
    cudaAccessPolicyWindow win{};
    std::vector<uint32_t> h_jbits;  // host copy of the junction bitmap (sharding)
    // decode (ids -> bytes): per-id LUT + byte blob, workspace
    uint32_t *d_vinfo = nullptr;
    uint8_t *d_vblob = nullptr;
    uint4 *d_vrec = nullptr;
    uint8_t *d_vlen = nullptr;
    uint32_t *d_vlong = nullptr;
    bool vocab_ext = false;  // decode vocabulary with empty or >= 255-byte strings
    uint32_t n_vocab_dec = 0;
    DevBuf dec_state, dec_status, dec_tiles;  // dec_tiles: tile byte totals + offsets (two-pass)
    // GPT-2 regex pre-tokenization (optional mode)
    uint8_t *d_pt_classes = nullptr;
    uint32_t pt_n_cps = 0;
    uint8_t pt_ascii[128] = {};
    uint32_t mode = 0;
    DevBuf pt_bits;
    const uint32_t *cur_pretok = nullptr;  // bits for the encode being launched
    unsigned int dec_epoch = 0;
    int dec_grid = 0, dec_rows_grid = 0;
    // workspace
    DevBuf ws_state, ws_status, ws_recs, ws_scratch, ws_tiles, ws_arena, ws_gscr, ws_glist;
    // host-buffer entry point: pinned (device-mapped) staging + device copy
    DevBuf io_dev;
    uint8_t *pin = nullptr;
    uint8_t *pin_dev = nullptr;  // device alias of pin (mapped)
    size_t pin_bytes = 0;
    bool state_fresh = false;  // h_state already holds the last encode's state
    cudaEvent_t io_ev[2] = {nullptr, nullptr};
    // streamed host encode (gpubpe_encode_host on large batches): two slots of
    // pinned staging, device input and mapped pinned output; H2D on s_copy
    struct StreamSlot {
        uint8_t *pin_in = nullptr;
        size_t pin_in_bytes = 0;
        uint8_t *pin_out = nullptr, *pin_out_dev = nullptr;
        size_t pin_out_bytes = 0;
        DevBuf dev_in, dev_out;
        cudaEvent_t ev_h2d = nullptr, ev_done = nullptr, ev_d2h = nullptr;
    } ss[2];
    cudaStream_t s_copy = nullptr, s_d2h = nullptr;
    bool defer_check = false;  // the caller checks EncodeState.overflow itself (streamed encode)
    // overlapped host encode: the kernel is enqueued before the input pieces;
    // each piece's arrival word is DMA'd (s_copy) after it
    unsigned int *d_arrive = nullptr;  // [ARRIVE_MAX] device words
    unsigned int *h_tag = nullptr;     // pinned source of the words' value
    unsigned int arrive_tag = 0;
    const unsigned int *cur_arrive = nullptr;  // for the encode being launched
    uint64_t cur_piece = 0;
    unsigned long long *dbg_buf = nullptr;  // GPUBPE_DEBUG & 8 timestamps
    StateMirror *h_mirror = nullptr, *d_mirror = nullptr;  // host calls: the kernel's results (mapped)
    StateMirror *cur_mirror = nullptr;                     // for the encode being launched
    unsigned long long mirror_tag = 0;                     // per host call
    std::chrono::steady_clock::time_point t_call;  // GPUBPE_HOSTTIME: gpubpe_encode entry
    int tl_n = 0;                                  // GPUBPE_HOSTTIME=2: piece events of this call
    cudaEvent_t *tl_ev = nullptr;
    EncodeState *h_state_ss = nullptr;  // pinned [2]: per-slot encode state
    uint64_t last_n_tiles = 0;
    uint32_t n_ids = 0;             // internal ids the tables cover
    DevBuf mt_offs, mt_counts;      // token-level merges (gpubpe_merge_tokens)
    uint64_t n_allocs = 0, alloc_mark = 0;  // buffers allocated (grow-only workspaces), mark at call entry
    bool host_call = false;                  // inside gpubpe_encode_host (its mark stands)
    unsigned int epoch = 0;
    uint64_t calls = 0;  // selects the EncodeState slot (two, alternating)
    EncodeState *h_state = nullptr;  // pinned
    std::string err;
    bool profiling = false;
    uint64_t last_n_bytes = 0;
    bool timed = false;  // events of the last encode are valid
    cudaEvent_t ev[2] = {nullptr, nullptr};
};

static int fail(gpubpe_ctx *c, int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->err = buf;
    return code;
}

#define CK(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return fail(ctx, e_ == cudaErrorMemoryAllocation ? GPUBPE_ENOMEM : GPUBPE_ECUDA, \
                        "%s: %s", #call, cudaGetErrorString(e_));                         \
    } while (0)

static size_t table_slot(size_t bytes) { return (std::max<size_t>(bytes, 16) + 255) & ~(size_t)255; }

template <typename V>
static int upload(gpubpe_ctx *ctx, const std::vector<V> &h, const V **out) {
    size_t bytes = table_slot(h.size() * sizeof(V));
    if (ctx->tables_used + bytes > ctx->tables_bytes)
        return fail(ctx, GPUBPE_ENOMEM, "table arena too small (%zu + %zu > %zu)", ctx->tables_used,
                    bytes, ctx->tables_bytes);
    uint8_t *d = ctx->tables + ctx->tables_used;
    ctx->tables_used += bytes;
    if (!h.empty()) CK(cudaMemcpy(d, h.data(), h.size() * sizeof(V), cudaMemcpyHostToDevice));
    *out = reinterpret_cast<const V *>(d);
    return GPUBPE_OK;
}

static int ensure(gpubpe_ctx *ctx, DevBuf &b, size_t bytes, bool zero) {
    if (b.bytes >= bytes && b.p) return GPUBPE_OK;
    CK(cudaDeviceSynchronize());
    if (b.p) CK(cudaFree(b.p));
    b.p = nullptr;
    b.bytes = 0;
    size_t nb = std::max<size_t>(bytes + bytes / 4, 256);
    CK(cudaMalloc(&b.p, nb));
    ++ctx->n_allocs;
    if (zero) CK(cudaMemset(b.p, 0, nb));
    b.bytes = nb;
    return GPUBPE_OK;
}

#ifndef GPUBPE_MEMO_SPREAD
#define GPUBPE_MEMO_SPREAD 8  // memo slots per string (power-of-two capacity): short probe chains
#endif

static uint64_t memo_hash_bytes(const uint8_t *s, uint32_t len) {
    uint64_t h = memo_hash_init(len);
    for (uint32_t c = 0; c < len || c == 0; c += 8) {
        uint64_t ch = 0;
        for (uint32_t j = c; j < len && j < c + 8; ++j) ch |= (uint64_t)s[j] << (8 * (j - c));
        h = memo_hash_step(h, ch);
        if (len <= 8) break;
    }
    return h;
}

static int encode_impl(gpubpe_ctx *ctx, const uint8_t *d_bytes, uint64_t n_bytes,
                       const int64_t *d_doc_offs, uint64_t n_docs, uint64_t max_seq_len,
                       uint64_t chunk_budget, uint32_t *d_out_ids, int64_t *d_out_offs,
                       cudaStream_t s, bool *checked);

// ctx_create phase timing (GPUBPE_HOSTTIME): stamp k at the start of phase k
#define BUILD_STAMP(k) (build_t[k] = std::chrono::steady_clock::now())

extern "C" __attribute__((visibility("default"))) int gpubpe_ctx_create(int device, const uint32_t *base_ids, const uint32_t *left,
                                 const uint32_t *right, const uint32_t *rank,
                                 const uint32_t *new_tok, uint64_t n_rules,
                                 const uint32_t *vocab_ids, const uint8_t *vocab_bytes,
                                 const uint64_t *vocab_offs, uint64_t n_vocab, uint32_t flags,
                                 gpubpe_ctx **out) {
    if (!out) return GPUBPE_EINVAL;
    *out = nullptr;
    std::chrono::steady_clock::time_point build_t[8];
    BUILD_STAMP(7);
    gpubpe_ctx *ctx = new gpubpe_ctx();
    *out = ctx;  // on failure the caller reads the message, then destroys
    ctx->device = device;
    ctx->flags = flags;
    int rc = GPUBPE_OK;
    auto bail = [&](int code) {
        *out = ctx;  // keep the message readable; caller destroys
        return code;
    };
    if (!base_ids || (n_rules && (!left || !right || !rank || !new_tok)))
        return bail(fail(ctx, GPUBPE_EINVAL, "null table pointer"));
    {
        cudaError_t e = cudaSetDevice(device);
        if (e != cudaSuccess) return bail(fail(ctx, GPUBPE_ECUDA, "cudaSetDevice(%d): %s", device, cudaGetErrorString(e)));
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        ctx->num_sms = sms;
        if ((e = setup_kernels()) != cudaSuccess)
            return bail(fail(ctx, GPUBPE_ECUDA, "kernel setup: %s", cudaGetErrorString(e)));
        // the per-lane engine keeps its token arrays on the thread stack
        size_t stack = 0;
        cudaDeviceGetLimit(&stack, cudaLimitStackSize);
        if (stack < 4096 && (e = cudaDeviceSetLimit(cudaLimitStackSize, 4096)) != cudaSuccess)
            return bail(fail(ctx, GPUBPE_ECUDA, "stack limit: %s", cudaGetErrorString(e)));
        int blocks = 0;
        if ((e = tile_occupancy(&blocks)) != cudaSuccess || blocks < 1)
            return bail(fail(ctx, GPUBPE_ECUDA, "encode kernel does not fit an SM (%d blocks, %s)", blocks,
                             cudaGetErrorString(e)));
        int coop = 0;
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
        if (!coop) return bail(fail(ctx, GPUBPE_ECUDA, "device %d lacks cooperative launch", device));
        ctx->tile_blocks_per_sm = blocks;
    }

    BUILD_STAMP(0);
    // ---- internal ids: used as-is when every id < 2^24, else densely remapped
    uint64_t max_id = 0;
    for (int b = 0; b < 256; ++b) max_id = std::max<uint64_t>(max_id, base_ids[b]);
    for (uint64_t i = 0; i < n_rules; ++i) {
        max_id = std::max<uint64_t>(max_id, left[i]);
        max_id = std::max<uint64_t>(max_id, right[i]);
        max_id = std::max<uint64_t>(max_id, new_tok[i]);
        if (rank[i] == GPUBPE_INF)
            return bail(fail(ctx, GPUBPE_EINVAL, "rule %llu: rank 0xFFFFFFFF is reserved", (unsigned long long)i));
    }
    const bool identity = max_id < (1ull << 24);
    std::unordered_map<uint32_t, uint32_t> remap;
    std::vector<uint32_t> ext;  // internal -> external
    auto intern = [&](uint32_t x) -> uint32_t {
        if (identity) return x;
        auto it = remap.find(x);
        if (it != remap.end()) return it->second;
        uint32_t v = (uint32_t)ext.size();
        remap.emplace(x, v);
        ext.push_back(x);
        return v;
    };
    std::vector<uint32_t> base(256), L(n_rules), R(n_rules), NW(n_rules);
    for (int b = 0; b < 256; ++b) base[b] = intern(base_ids[b]);
    for (uint64_t i = 0; i < n_rules; ++i) {
        L[i] = intern(left[i]);
        R[i] = intern(right[i]);
        NW[i] = intern(new_tok[i]);
    }
    const uint64_t n_ids = identity ? max_id + 1 : ext.size();
    if (n_ids >= (1ull << 24))
        return bail(fail(ctx, GPUBPE_EINVAL, "more than 2^24 distinct token ids (%llu)", (unsigned long long)n_ids));

    BUILD_STAMP(1);
    // ---- pair table: two-choice cuckoo (common.cuh pair_slots) at <= 50% load;
    //      an insertion that cannot settle doubles the capacity and starts over
    uint64_t cap = 2;
    while (cap < 2 * n_rules) cap <<= 1;
    std::vector<uint4> slots;
    for (;;) {
        slots.assign(cap, make_uint4(GPUBPE_INF, GPUBPE_INF, 0, 0));
        const uint32_t mask = (uint32_t)(cap - 1);
        auto empty = [](const uint4 &v) { return v.x == GPUBPE_INF && v.y == GPUBPE_INF; };
        bool settled = true;
        for (uint64_t i = 0; i < n_rules && settled; ++i) {
            const PairSlots ps = pair_slots(L[i], R[i], mask);
            for (uint32_t h : {ps.a, ps.b})
                if (slots[h].x == L[i] && slots[h].y == R[i])
                    return bail(fail(ctx, GPUBPE_ETABLE, "pair (%u, %u) duplicated at rank %u",
                                     left[i], right[i], rank[i]));
            uint4 cur = make_uint4(L[i], R[i], rank[i], NW[i]);
            uint32_t pos = empty(slots[ps.a]) || !empty(slots[ps.b]) ? ps.a : ps.b;
            for (int kick = 0;; ++kick) {
                if (empty(slots[pos])) {
                    slots[pos] = cur;
                    break;
                }
                if (kick == 512) {
                    settled = false;
                    break;
                }
                std::swap(cur, slots[pos]);  // the evicted rule moves to its other slot
                const PairSlots q = pair_slots(cur.x, cur.y, mask);
                pos = pos == q.a ? q.b : q.a;
            }
        }
        if (settled) break;
        cap <<= 1;
    }
    BUILD_STAMP(2);
    // ---- rl / rr and well-formedness
    // one extra entry: id n_ids is an inert sentinel no rule mentions (token-level
    // callers map ids outside the table to it, gpubpe_merge_tokens)
    std::vector<uint32_t> rl(n_ids + 1, GPUBPE_INF), rr(n_ids + 1, GPUBPE_INF);
    std::vector<int64_t> maxprod(n_ids, -1);
    for (uint64_t i = 0; i < n_rules; ++i) {
        rl[L[i]] = std::min(rl[L[i]], rank[i]);
        rr[R[i]] = std::min(rr[R[i]], rank[i]);
        maxprod[NW[i]] = std::max<int64_t>(maxprod[NW[i]], rank[i]);
    }
    bool wf = !(flags & GPUBPE_F_STRICT);
    for (uint64_t i = 0; i < n_rules && wf; ++i)  // the warp engine packs ranks into 31 bits
        if (rank[i] >= 0x7FFFFFFFu) wf = false;
    for (uint64_t i = 0; i < n_rules && wf; ++i)
        if ((int64_t)rank[i] <= maxprod[L[i]] || (int64_t)rank[i] <= maxprod[R[i]]) wf = false;
    BUILD_STAMP(3);
    // ---- junction bitmap: first/last covered byte sets to a fixpoint; built on
    //      the device (build.cu) unless GPUBPE_F_HOST_TABLES asks for the host loops
    std::vector<uint32_t> jbits(2048);
    if (!(flags & GPUBPE_F_HOST_TABLES)) {
        int rounds = 0;
        cudaError_t e = build_junction_device(base.data(), L.data(), R.data(), NW.data(), n_rules, n_ids,
                                              jbits.data(), &rounds);
        if (e != cudaSuccess)
            return bail(fail(ctx, GPUBPE_ECUDA, "junction build: %s", cudaGetErrorString(e)));
    } else {
        std::vector<uint64_t> F(n_ids * 4, 0), B(n_ids * 4, 0);
        for (int b = 0; b < 256; ++b) {
            F[base[b] * 4 + (b >> 6)] |= 1ull << (b & 63);
            B[base[b] * 4 + (b >> 6)] |= 1ull << (b & 63);
        }
        std::vector<uint64_t> order(n_rules);
        for (uint64_t i = 0; i < n_rules; ++i) order[i] = i;
        std::sort(order.begin(), order.end(), [&](uint64_t x, uint64_t y) { return rank[x] < rank[y]; });
        for (bool changed = true; changed;) {
            changed = false;
            for (uint64_t oi : order) {
                for (int w = 0; w < 4; ++w) {
                    uint64_t f = F[NW[oi] * 4 + w] | F[L[oi] * 4 + w];
                    uint64_t l = B[NW[oi] * 4 + w] | B[R[oi] * 4 + w];
                    if (f != F[NW[oi] * 4 + w] || l != B[NW[oi] * 4 + w]) changed = true;
                    F[NW[oi] * 4 + w] = f;
                    B[NW[oi] * 4 + w] = l;
                }
            }
        }
        std::vector<uint64_t> J(65536 / 64, 0);  // row x: 256 bits of y
        for (uint64_t i = 0; i < n_rules; ++i) {
            for (int x = 0; x < 256; ++x) {
                if (!((B[L[i] * 4 + (x >> 6)] >> (x & 63)) & 1)) continue;
                for (int w = 0; w < 4; ++w) J[x * 4 + w] |= F[R[i] * 4 + w];
            }
        }
        for (int k = 0; k < 2048; ++k) jbits[k] = (uint32_t)(J[k >> 1] >> (32 * (k & 1)));
    }
    ctx->h_jbits = jbits;

    // memo upper bounds (the memo is built after a verification encode)
    uint64_t memo_cand = 0, blob_max = 0;
    if (!(flags & GPUBPE_F_NO_MEMO) && n_vocab && vocab_ids && vocab_bytes && vocab_offs)
        for (uint64_t v = 0; v < n_vocab; ++v) {
            uint64_t len = vocab_offs[v + 1] - vocab_offs[v];
            if (len < 2 || len > SHORT_MAX) continue;
            ++memo_cand;
            if (len > 8) blob_max += (len - 1) / 8 * 8;
        }
    uint64_t memo_cap_max = 2;
    while (memo_cap_max < (uint64_t)GPUBPE_MEMO_SPREAD * memo_cand) memo_cap_max <<= 1;
    {
        size_t need = table_slot(slots.size() * sizeof(uint4)) + 2 * table_slot((n_ids + 1) * 4) +
                      table_slot(jbits.size() * 4) + table_slot(256 * 4) +
                      (identity ? 0 : table_slot(ext.size() * 4)) +
                      table_slot(memo_cap_max * sizeof(uint4)) + table_slot(blob_max);
        void *d = nullptr;
        cudaError_t e = cudaMalloc(&d, need);
        if (e != cudaSuccess) return bail(fail(ctx, GPUBPE_ENOMEM, "tables (%zu B): %s", need, cudaGetErrorString(e)));
        ctx->tables = static_cast<uint8_t *>(d);
        ctx->tables_bytes = need;
    }
    const uint32_t *d_rl, *d_rr, *d_j, *d_base;
    const uint4 *d_pairs;
    if ((rc = upload(ctx, slots, &d_pairs))) return bail(rc);
    if ((rc = upload(ctx, rl, &d_rl))) return bail(rc);
    if ((rc = upload(ctx, rr, &d_rr))) return bail(rc);
    if ((rc = upload(ctx, jbits, &d_j))) return bail(rc);
    if ((rc = upload(ctx, base, &d_base))) return bail(rc);
    ctx->T.pairs = d_pairs;
    ctx->T.pair_mask = (uint32_t)(cap - 1);
    ctx->T.rl = d_rl;
    ctx->T.rr = d_rr;
    ctx->T.jbits = d_j;
    ctx->T.base = d_base;
    ctx->T.memo = nullptr;
    ctx->T.memo_mask = 0;
    ctx->T.blob = nullptr;
    ctx->T.well_formed = wf ? 1 : 0;
    ctx->n_ids = (uint32_t)n_ids;
    ctx->T.ext_id = nullptr;
    if (!identity) {
        const uint32_t *d_ext;
        if ((rc = upload(ctx, ext, &d_ext))) return bail(rc);
        ctx->T.ext_id = d_ext;
    }
    ctx->h_state = nullptr;
    {
        cudaError_t e = cudaMallocHost(&ctx->h_state, sizeof(EncodeState));
        (void)0;
        if (e != cudaSuccess) return bail(fail(ctx, GPUBPE_ENOMEM, "pinned state: %s", cudaGetErrorString(e)));
        memset(ctx->h_state, 0, sizeof(EncodeState));
    }

    BUILD_STAMP(4);
    // ---- memo: vocab strings whose BPE (computed by this engine) is themselves
    if (!(flags & GPUBPE_F_NO_MEMO) && n_vocab && vocab_ids && vocab_bytes && vocab_offs) {
        std::vector<uint64_t> cand;
        std::vector<uint32_t> cand_int;
        for (uint64_t v = 0; v < n_vocab; ++v) {
            uint64_t len = vocab_offs[v + 1] - vocab_offs[v];
            if (len < 2 || len > SHORT_MAX) continue;
            uint32_t id = vocab_ids[v];
            uint32_t iid;
            if (identity) {
                if (id >= n_ids) continue;
                iid = id;
            } else {
                auto it = remap.find(id);
                if (it == remap.end()) continue;
                iid = it->second;
            }
            cand.push_back(v);
            cand_int.push_back(iid);
        }
        if (!cand.empty()) {
            std::vector<uint8_t> hb;
            std::vector<int64_t> ho(cand.size() + 1, 0);
            for (size_t k = 0; k < cand.size(); ++k) {
                uint64_t v = cand[k];
                hb.insert(hb.end(), vocab_bytes + vocab_offs[v], vocab_bytes + vocab_offs[v + 1]);
                ho[k + 1] = (int64_t)hb.size();
            }
            uint8_t *db = nullptr;
            int64_t *dof = nullptr, *doo = nullptr;
            uint32_t *dids = nullptr;
            CK(cudaMalloc(&db, hb.size()));
            CK(cudaMalloc(&dof, ho.size() * 8));
            CK(cudaMalloc(&doo, ho.size() * 8));
            CK(cudaMalloc(&dids, hb.size() * 4));
            CK(cudaMemcpy(db, hb.data(), hb.size(), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(dof, ho.data(), ho.size() * 8, cudaMemcpyHostToDevice));
            DevTables saved = ctx->T;
            ctx->T.ext_id = nullptr;  // verify in internal ids
            bool checked = false;
            rc = encode_impl(ctx, db, hb.size(), dof, cand.size(), ~0ull >> 2, ~0ull >> 2, dids,
                             doo, 0, &checked);
            ctx->T = saved;
            if (rc) return bail(rc);
            CK(cudaDeviceSynchronize());
            std::vector<int64_t> oo(ho.size());
            std::vector<uint32_t> oids(hb.size());
            CK(cudaMemcpy(oo.data(), doo, oo.size() * 8, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(oids.data(), dids, hb.size() * 4, cudaMemcpyDeviceToHost));
            cudaFree(db); cudaFree(dof); cudaFree(doo); cudaFree(dids);
            std::vector<size_t> keep;
            for (size_t k = 0; k < cand.size(); ++k)
                if (oo[k + 1] - oo[k] == 1 && oids[oo[k]] == cand_int[k]) keep.push_back(k);
            uint64_t mcap = 2;
            while (mcap < (size_t)GPUBPE_MEMO_SPREAD * keep.size()) mcap <<= 1;  // load <= 1 / spread
            std::vector<uint4> memo(mcap, make_uint4(0, 0, 0, 0));
            std::vector<unsigned long long> blob;  // bytes 8.. as zero-padded 8-byte chunks
            for (size_t k : keep) {
                const uint8_t *sv = hb.data() + ho[k];
                uint32_t len = (uint32_t)(ho[k + 1] - ho[k]);
                uint64_t lo = 0;
                for (uint32_t j = 0; j < len && j < 8; ++j) lo |= (uint64_t)sv[j] << (8 * j);
                uint32_t boff = (uint32_t)blob.size();
                if (len > 8) {
                    if (boff >= (1u << 24)) continue;  // blob offset field is 24 bits
                    for (uint32_t c = 8; c < len; c += 8) {
                        unsigned long long ch = 0;
                        for (uint32_t j = c; j < len && j < c + 8; ++j) ch |= (unsigned long long)sv[j] << (8 * (j - c));
                        blob.push_back(ch);
                    }
                }
                uint32_t h = memo_slot_of(memo_hash_bytes(sv, len), (uint32_t)(mcap - 1));
                while (memo[h].w != 0) h = (h + 1) & (uint32_t)(mcap - 1);
                memo[h] = make_uint4((uint32_t)lo, (uint32_t)(lo >> 32), cand_int[k],
                                     len | (len > 8 ? boff << 8 : 0u));
            }
            const uint4 *d_memo;
            const unsigned long long *d_blob;
            if ((rc = upload(ctx, memo, &d_memo))) return bail(rc);
            if ((rc = upload(ctx, blob, &d_blob))) return bail(rc);
            ctx->T.memo = d_memo;
            ctx->T.memo_mask = (uint32_t)(mcap - 1);
            ctx->T.blob = d_blob;
        }
    }
    BUILD_STAMP(5);
    // ---- keep the tables resident in L2 across unrelated traffic
    {
        int persist_max = 0, win_max = 0;
        cudaDeviceGetAttribute(&persist_max, cudaDevAttrMaxPersistingL2CacheSize, device);
        cudaDeviceGetAttribute(&win_max, cudaDevAttrMaxAccessPolicyWindowSize, device);
        size_t want = std::min<size_t>(ctx->tables_used, (size_t)persist_max);
        size_t cur = 0;
        cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
        if (want > cur) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
        cudaGetLastError();
        size_t win = std::min<size_t>(ctx->tables_used, (size_t)win_max);
        if (want && win) {
            ctx->win.base_ptr = ctx->tables;
            ctx->win.num_bytes = win;
            ctx->win.hitRatio = std::min(1.0f, (float)want / (float)win);
            ctx->win.hitProp = cudaAccessPropertyPersisting;
            ctx->win.missProp = cudaAccessPropertyStreaming;
        }
    }
    *out = ctx;
    if (getenv("GPUBPE_HOSTTIME")) {
        auto ms = [&](int a, int b) { return std::chrono::duration<double, std::milli>(build_t[b] - build_t[a]).count(); };
        const auto end = std::chrono::steady_clock::now();
        fprintf(stderr, "ctx_create: setup %.1f | intern %.1f | pairs %.1f | rl/rr %.1f | junction %.1f | memo %.1f | l2 %.1f ms\n",
                ms(7, 0), ms(0, 1), ms(1, 2), ms(2, 3), ms(3, 4), ms(4, 5),
                std::chrono::duration<double, std::milli>(end - build_t[5]).count());
    }
    return GPUBPE_OK;
}

// Debug timestamps of the last encode (GPUBPE_DEBUG & 8) to GPUBPE_DEBUG_OUT.
static void dump_debug(gpubpe_ctx *ctx, cudaStream_t s) {
    const char *path = getenv("GPUBPE_DEBUG_OUT");
    if (!path || !*path || !ctx->dbg_buf) return;
    std::vector<unsigned long long> h(40960);
    cudaMemcpyAsync(h.data(), ctx->dbg_buf, h.size() * 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    FILE *f = fopen(path, "wb");
    if (f) {
        fwrite(h.data(), 8, h.size(), f);
        fclose(f);
    }
}

static int encode_impl(gpubpe_ctx *ctx, const uint8_t *d_bytes, uint64_t n_bytes,
                       const int64_t *d_doc_offs, uint64_t n_docs, uint64_t max_seq_len,
                       uint64_t chunk_budget, uint32_t *d_out_ids, int64_t *d_out_offs,
                       cudaStream_t s, bool *checked) {
    *checked = false;
    // one CTA of NW autonomous warps per SM, all co-resident (cooperative)
    const int grid = ctx->num_sms * ctx->tile_blocks_per_sm;
    // tile width: the largest of 512/256/128 bytes that still gives every
    // warp of the grid two tiles (small inputs get more, smaller tiles)
    const uint64_t n_warps = (uint64_t)grid * NW;
    int wt = 128;
    if (n_bytes >= 2 * n_warps * 512) wt = 512;
    else if (n_bytes >= 2 * n_warps * 256) wt = 256;
    if (const char *e = getenv("GPUBPE_WT")) {  // tuning override: 128, 256 or 512
        const int w = atoi(e);
        if (w == 128 || w == 256 || w == 512) wt = w;
    }
    const uint64_t n_tiles = (n_bytes + wt - 1) / wt;
    const uint64_t R = std::min<uint64_t>(n_tiles, (uint64_t)UNIT_MAX * grid);
    const uint64_t n_rounds = (n_tiles + R - 1) / R;
    // deferred segments (> SHORT_MAX bytes) start at least SHORT_MAX + 1 apart
    const uint64_t def_max = n_bytes / (SHORT_MAX + 1) + 1;
    int rc;
    if ((rc = ensure(ctx, ctx->ws_state, 2 * sizeof(EncodeState), true))) return rc;
    const uint64_t n_units = n_rounds * grid;
    if (ctx->ws_status.bytes < n_units * 8) ctx->epoch = 0;
    if ((rc = ensure(ctx, ctx->ws_status, n_units * 8, true))) return rc;
    if ((rc = ensure(ctx, ctx->ws_scratch, 2 * R * SLOT * 4, false))) return rc;
    if ((rc = ensure(ctx, ctx->ws_tiles, 2 * R * 8, false))) return rc;
    if ((rc = ensure(ctx, ctx->ws_recs, std::max<uint64_t>(1 << 16, std::min<uint64_t>(def_max, 1 << 20)) * sizeof(DefRec), false))) return rc;
    if ((rc = ensure(ctx, ctx->ws_arena, 64ull << 20, false))) return rc;
    if ((rc = ensure(ctx, ctx->ws_gscr, (8 + 2 * (size_t)grid) * 8, false))) return rc;
    for (int attempt = 0; attempt < 4; ++attempt) {
        const uint64_t rec_cap = ctx->ws_recs.bytes / sizeof(DefRec);
        if ((rc = ensure(ctx, ctx->ws_glist, rec_cap * 4, false))) return rc;
        if (++ctx->epoch >= (1u << 20)) {
            CK(cudaMemsetAsync(ctx->ws_status.p, 0, ctx->ws_status.bytes, s));
            ctx->epoch = 1;
        }
        EncodeState *slots = static_cast<EncodeState *>(ctx->ws_state.p);
        const uint64_t k = ctx->calls++;
        EncodeParams P{};
        P.T = ctx->T;
        P.bytes = d_bytes;
        P.n_bytes = n_bytes;
        P.doc_offs = reinterpret_cast<const long long *>(d_doc_offs);
        P.n_docs = n_docs;
        P.max_seq_len = max_seq_len;
        P.chunk_budget = chunk_budget;
        P.out_ids = d_out_ids;
        P.out_offs = reinterpret_cast<long long *>(d_out_offs);
        P.st = slots + (k & 1);
        P.st_next = slots + ((k + 1) & 1);
        P.scratch = static_cast<uint32_t *>(ctx->ws_scratch.p);
        P.tiles = static_cast<unsigned long long *>(ctx->ws_tiles.p);
        P.status = static_cast<unsigned long long *>(ctx->ws_status.p);
        P.recs = static_cast<DefRec *>(ctx->ws_recs.p);
        P.rec_cap = rec_cap;
        P.arena = static_cast<uint32_t *>(ctx->ws_arena.p);
        P.arena_words = ctx->ws_arena.bytes / 4;
        P.n_tiles = n_tiles;
        P.round_tiles = R;
        P.epoch = ctx->epoch;
        P.strict = (ctx->flags & GPUBPE_F_STRICT) ? 1 : 0;
        P.aligned = (reinterpret_cast<uintptr_t>(d_bytes) & 15) == 0;
        P.tile_bytes = wt;
        P.pretok = ctx->cur_pretok;
        P.arrive = ctx->cur_arrive;
        P.piece = ctx->cur_piece ? ctx->cur_piece : 1;
        P.arrive_tag = ctx->arrive_tag;
        P.mirror = ctx->cur_mirror;
        P.mirror_tag = ctx->mirror_tag;
        P.gscr = static_cast<unsigned long long *>(ctx->ws_gscr.p);
        P.glist = static_cast<uint32_t *>(ctx->ws_glist.p);
        ctx->last_n_tiles = n_tiles;
        // debug knobs (tuning only) never apply to the memo verification encode
        const int dbg = (ctx->T.memo && getenv("GPUBPE_DEBUG")) ? atoi(getenv("GPUBPE_DEBUG")) : 0;
        P.dbg_phase_a_only = (dbg & 16) ? 1 : (dbg & 32) ? 2 : 0;
        if (dbg & 8) {
            if (!ctx->dbg_buf) cudaMalloc(&ctx->dbg_buf, 40960 * 8);
            cudaMemsetAsync(ctx->dbg_buf, 0, 40960 * 8, s);
            P.dbg = ctx->dbg_buf;
        }
        static const bool htime_l = getenv("GPUBPE_HOSTTIME") != nullptr;
        const auto tl0 = std::chrono::steady_clock::now();
        cudaError_t e = launch_encode(P, grid, s, ctx->profiling ? ctx->ev : nullptr, (dbg & 4) ? nullptr : &ctx->win, !(dbg & 2));
        if (htime_l)
            fprintf(stderr, "encode_impl: setup %.1f | launch %.1f us\n",
                    std::chrono::duration<double, std::micro>(tl0 - ctx->t_call).count(),
                    std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - tl0).count());
        ctx->timed = ctx->profiling;
        if (e != cudaSuccess) return fail(ctx, GPUBPE_ECUDA, "encode launch: %s", cudaGetErrorString(e));
        // Overflow is impossible when every deferred segment fits the record
        // list and the arena (ENGINE_BYTES(len) rounded to 16 B per segment);
        // otherwise check after the call and re-run with larger buffers.
        const uint64_t arena_need = 26 * n_bytes + 96 * def_max;
        if ((dbg & 8) && !P.arrive) dump_debug(ctx, s);  // (overlapped calls: after their pieces)
        if (ctx->defer_check || (def_max <= rec_cap && arena_need <= ctx->ws_arena.bytes)) return GPUBPE_OK;
        *checked = true;
        CK(cudaMemcpyAsync(ctx->h_state, P.st, sizeof(EncodeState), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (!ctx->h_state->overflow) return GPUBPE_OK;
        const uint64_t nd = ctx->h_state->bar >> 32;
        if (nd > rec_cap && (rc = ensure(ctx, ctx->ws_recs, nd * sizeof(DefRec), false))) return rc;
        const uint64_t used = ctx->h_state->arena_used * 4;
        if (used > ctx->ws_arena.bytes && (rc = ensure(ctx, ctx->ws_arena, used, false))) return rc;
    }
    return fail(ctx, GPUBPE_ENOMEM, "deferred-segment buffers kept overflowing");
}

extern "C" __attribute__((visibility("default"))) int gpubpe_encode(gpubpe_ctx *ctx, const uint8_t *d_bytes, uint64_t n_bytes,
                             const int64_t *d_doc_offs, uint64_t n_docs, uint64_t max_seq_len,
                             uint64_t chunk_budget, uint32_t *d_out_ids, int64_t *d_out_offs,
                             void *stream) {
    if (!ctx) return GPUBPE_EINVAL;
    ctx->t_call = std::chrono::steady_clock::now();
    if (chunk_budget < 2 || chunk_budget > max_seq_len)
        return fail(ctx, GPUBPE_EINVAL, "chunk_budget must be in [2, max_seq_len]");
    if (n_docs && (!d_doc_offs || !d_out_offs)) return fail(ctx, GPUBPE_EINVAL, "null offsets");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!ctx->host_call) ctx->alloc_mark = ctx->n_allocs;
    CK(cudaSetDevice(ctx->device));
    ctx->state_fresh = false;
    ctx->last_n_bytes = n_docs ? n_bytes : 0;
    ctx->timed = false;
    if (n_bytes == 0 || n_docs == 0) {
        if (n_docs) CK(cudaMemsetAsync(d_out_offs, 0, (n_docs + 1) * 8, s));
        int rc = ensure(ctx, ctx->ws_state, 2 * sizeof(EncodeState), true);
        if (rc) return rc;
        const uint64_t k = ctx->calls++;
        CK(cudaMemsetAsync(static_cast<EncodeState *>(ctx->ws_state.p) + (k & 1), 0, sizeof(EncodeState), s));
        CK(cudaMemsetAsync(static_cast<EncodeState *>(ctx->ws_state.p) + ((k + 1) & 1), 0, sizeof(EncodeState), s));
        return GPUBPE_OK;
    }
    if (!d_bytes || !d_out_ids) return fail(ctx, GPUBPE_EINVAL, "null data pointer");
    const uint32_t *pt = nullptr;
    if (ctx->mode == GPUBPE_MODE_GPT2_REGEX) {  // pre-token starts, then the same encode
        const uint64_t n_words = (n_bytes + 31) / 32;
        int rc2;
        if ((rc2 = ensure(ctx, ctx->pt_bits, (n_words + 64) * 4, false))) return rc2;
        PretokParams Q{};
        Q.bytes = d_bytes;
        Q.n_bytes = n_bytes;
        Q.doc_offs = reinterpret_cast<const long long *>(d_doc_offs);
        Q.n_docs = n_docs;
        Q.classes = ctx->d_pt_classes;
        Q.n_cps = ctx->pt_n_cps;
        memcpy(Q.ascii, ctx->pt_ascii, 128);
        Q.ascii_std = 1;
        Q.paths = getenv("GPUBPE_PRETOK_PATHS") ? (uint32_t)atoi(getenv("GPUBPE_PRETOK_PATHS")) : 7u;  // (tests)
        for (int c = 0; c < 128; ++c) {
            const uint8_t want = ((c | 32) >= 'a' && (c | 32) <= 'z') ? 1 : (c >= '0' && c <= '9') ? 2
                                 : ((c >= 9 && c <= 13) || c == ' ') ? 3 : 0;
            if (ctx->pt_ascii[c] != want) Q.ascii_std = 0;
        }
        Q.out = static_cast<uint32_t *>(ctx->pt_bits.p);
        Q.n_words = n_words;
        CK(cudaMemsetAsync(Q.out + n_words, 0, 64 * 4, s));  // halo words past the end
        CK(launch_pretok(Q, s));
        pt = Q.out;
    }
    ctx->cur_pretok = pt;
    bool checked;
    return encode_impl(ctx, d_bytes, n_bytes, d_doc_offs, n_docs, max_seq_len, chunk_budget,
                       d_out_ids, d_out_offs, s, &checked);
}

// Host cores this process may use for its copy threads: the machine's, divided
// among the ranks of one node (LOCAL_WORLD_SIZE, set by torchrun), at least 2.
static unsigned host_cores_per_process() {
    const unsigned hw = std::max(2u, std::thread::hardware_concurrency());
    const char *lw = getenv("LOCAL_WORLD_SIZE");
    const unsigned ranks = lw ? (unsigned)std::max(1, atoi(lw)) : 1u;
    return std::max(2u, hw / ranks);
}

// Host copies through pinned memory (staging, copy-out) on a small persistent
// worker pool: the caller copies one chunk itself, workers the others.
namespace {
class CopyPool {
  public:
    static CopyPool &get() {
        static CopyPool *p = new CopyPool();  // never destroyed: workers live for the process
        return *p;
    }
    unsigned workers() const { return (unsigned)th_.size(); }
    // Runs part(0) .. part(parts - 1): the caller takes part 0 and whatever the
    // workers have not picked up when it is done, then waits for the rest.
    void run(unsigned parts, const std::function<void(unsigned)> &part) {
        {
            std::lock_guard<std::mutex> g(m_);
            for (unsigned i = 1; i < parts; ++i) {
                jobs_.push_back([&part, i] { part(i); });
                ++pending_;
            }
        }
        cv_.notify_all();
        part(0);
        for (;;) {
            std::function<void()> j;
            {
                std::unique_lock<std::mutex> g(m_);
                if (jobs_.empty()) {
                    done_.wait(g, [&] { return pending_ == 0; });
                    return;
                }
                j = std::move(jobs_.back());
                jobs_.pop_back();
            }
            j();
            finish();
        }
    }

  private:
    CopyPool() {
        const unsigned hw = host_cores_per_process();
        const unsigned nw = std::min(7u, hw - 1);
        for (unsigned i = 0; i < nw; ++i) th_.emplace_back([this] { loop(); });
        for (auto &t : th_) t.detach();
    }
    void finish() {
        std::lock_guard<std::mutex> g(m_);
        if (--pending_ == 0) done_.notify_all();
    }
    void loop() {
        for (;;) {
            std::function<void()> j;
            {
                std::unique_lock<std::mutex> g(m_);
                cv_.wait(g, [&] { return !jobs_.empty(); });
                j = std::move(jobs_.back());
                jobs_.pop_back();
            }
            j();
            finish();
        }
    }
    std::vector<std::thread> th_;
    std::mutex m_;
    std::condition_variable cv_, done_;
    std::vector<std::function<void()>> jobs_;
    size_t pending_ = 0;
};
}  // namespace

// Staging helpers for the latency path: a few workers that are woken when a
// host call begins and spin for work only while one is active, so the
// piecewise staging copies of a ~0.5 MiB batch split across cores without a
// thread wake-up per copy (and without spinning between calls).
static inline void cpu_relax() {
#if defined(__x86_64__) || defined(__i386__)
    __builtin_ia32_pause();
#endif
}

// Copies bytes [lo, hi) of the batch to dst (gather entry point: documents
// in separate buffers); null for a contiguous h_bytes.
using StageFn = std::function<void(uint8_t *dst, uint64_t lo, uint64_t hi)>;

namespace {
// Jobs: a buffer split in parts (at most 40).  One 64-bit word holds the job
// id, its part count and the claimed parts, so a claim (CAS) can only succeed
// on the job it read, and a job's buffers are only rewritten once all its
// parts are done (left_ == 0) -- no part is ever run with another job's buffers.
class StagePool {
  public:
    static StagePool &get() {
        static StagePool *p = new StagePool();  // never destroyed: workers live for the process
        return *p;
    }
    void begin() {
        if (active_.fetch_add(1) == 0 && sleeping_.load(std::memory_order_acquire) > 0) {
            std::lock_guard<std::mutex> g(m_);
            cv_.notify_all();
        }
    }
    void end() {
        last_end_.store(now_ns(), std::memory_order_relaxed);
        active_.fetch_sub(1, std::memory_order_release);
    }
    // memcpy split in (workers + 1) parts, the caller working too
    void copy(uint8_t *dst, const uint8_t *src, size_t n) {
        const unsigned parts = (unsigned)th_.size() + 1;
        const size_t chunk = ((n + parts - 1) / parts + 63) & ~(size_t)63;
        // one staged job at a time; a concurrent caller (another context or
        // thread, e.g. one per GPU) copies its piece itself instead of waiting
        std::unique_lock<std::mutex> call(call_, std::try_to_lock);
        if (!call.owns_lock()) {
            memcpy(dst, src, n);
            return;
        }
        post(dst, src, n, chunk, parts);
        while (claim_and_run()) {
        }
        while (left_.load(std::memory_order_acquire) > 0) cpu_relax();
    }
    // the same for a gather: bytes [lo, hi) of the batch staged by fn, split in parts
    void gather(uint8_t *dst, const StageFn &fn, uint64_t lo, uint64_t hi) {
        const size_t n = hi - lo;
        const unsigned parts = (unsigned)th_.size() + 1;
        const size_t chunk = ((n + parts - 1) / parts + 63) & ~(size_t)63;
        std::unique_lock<std::mutex> call(call_, std::try_to_lock);
        if (!call.owns_lock()) {
            fn(dst, lo, hi);
            return;
        }
        fn_ = &fn;
        base_ = lo;
        post(dst, nullptr, n, chunk, parts);
        while (claim_and_run()) {
        }
        while (left_.load(std::memory_order_acquire) > 0) cpu_relax();
        fn_ = nullptr;
    }

  private:
    static constexpr unsigned MAXP = 40;
    static constexpr unsigned long long BITS = (1ull << MAXP) - 1;
    StagePool() {
        const unsigned hw = host_cores_per_process();
        const unsigned nw = std::min(7u, hw / 2 > 0 ? hw / 2 - 1 : 0u);  // host copies scale to ~8 threads
        for (unsigned i = 0; i < nw; ++i) th_.emplace_back([this] { loop(); });
        for (auto &t : th_) t.detach();
    }
    void post(uint8_t *dst, const uint8_t *src, size_t n, size_t chunk, unsigned parts) {
        dst_ = dst;
        src_ = src;
        n_ = n;
        chunk_ = chunk;
        left_.store((int)parts, std::memory_order_relaxed);
        job_ = (job_ + 1) & 0xFFFF;
        word_.store(((unsigned long long)job_ << 48) | ((unsigned long long)parts << 40), std::memory_order_release);
        gen_.fetch_add(1, std::memory_order_release);
    }
    // Claim and copy one part of the posted job; false when none is left.
    bool claim_and_run() {
        unsigned long long w = word_.load(std::memory_order_acquire);
        for (;;) {
            const unsigned parts = (unsigned)((w >> 40) & 0xFF);
            const unsigned long long free = ~w & BITS & ((1ull << parts) - 1);
            if (!free) return false;
            const unsigned i = (unsigned)__builtin_ctzll(free);
            if (word_.compare_exchange_weak(w, w | (1ull << i), std::memory_order_acq_rel,
                                            std::memory_order_acquire)) {
                const size_t lo = std::min(n_, i * chunk_), hi = std::min(n_, lo + chunk_);
                if (lo < hi) {
                    if (fn_) (*fn_)(dst_ + lo, base_ + lo, base_ + hi);
                    else memcpy(dst_ + lo, src_ + lo, hi - lo);
                }
                left_.fetch_sub(1, std::memory_order_acq_rel);
                return true;
            }
        }
    }
    static unsigned long long now_ns() {
        return (unsigned long long)std::chrono::duration_cast<std::chrono::nanoseconds>(
                   std::chrono::steady_clock::now().time_since_epoch()).count();
    }
    // Workers spin inside host calls and for a grace period after the last one
    // (GPUBPE_SPIN_US, default 200 us), so back-to-back calls find them awake
    // (a condition-variable wake-up costs several microseconds); then they sleep.
    void loop() {
        static const unsigned long long grace =
            1000ull * (unsigned long long)(getenv("GPUBPE_SPIN_US") ? atoll(getenv("GPUBPE_SPIN_US")) : 200);
        unsigned long long seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> g(m_);
                sleeping_.fetch_add(1);
                cv_.wait(g, [&] { return active_.load() > 0; });
                sleeping_.fetch_sub(1);
            }
            for (unsigned spins = 0;; ++spins) {
                if (active_.load(std::memory_order_acquire) == 0 && (spins & 1023) == 0 &&
                    now_ns() - last_end_.load(std::memory_order_relaxed) > grace)
                    break;
                const unsigned long long gen = gen_.load(std::memory_order_acquire);
                if (gen == seen) {
                    cpu_relax();
                    continue;
                }
                seen = gen;
                while (claim_and_run()) {
                }
            }
        }
    }
    std::vector<std::thread> th_;
    std::mutex m_, call_;
    std::condition_variable cv_;
    std::atomic<int> active_{0}, left_{0}, sleeping_{0};
    std::atomic<unsigned long long> word_{0}, gen_{0}, last_end_{0};
    unsigned job_ = 0;
    uint8_t *dst_ = nullptr;
    const uint8_t *src_ = nullptr;
    const StageFn *fn_ = nullptr;  // gather jobs: the stage function (else a memcpy from src_)
    uint64_t base_ = 0;            // gather jobs: batch offset of dst_
    size_t n_ = 0, chunk_ = 0;
};
}  // namespace

static void copy_par(void *dst, const void *src, size_t n) {
    const size_t per = 4u << 20;  // one chunk per 4 MiB beyond 8 MiB (below, a worker wake-up costs more)
    if (n <= 2 * per) {
        memcpy(dst, src, n);
        return;
    }
    CopyPool &pool = CopyPool::get();
    const unsigned parts = (unsigned)std::min<size_t>(pool.workers() + 1, (n + per - 1) / per);
    const size_t chunk = (n + parts - 1) / parts;
    pool.run(parts, [&](unsigned i) {
        const size_t lo = i * chunk, hi = std::min(n, lo + chunk);
        if (lo < hi) memcpy(static_cast<uint8_t *>(dst) + lo, static_cast<const uint8_t *>(src) + lo, hi - lo);
    });
}

// Gather documents (ptrs[d], lens[d]) back to back into dst (offs = their
// prefix sums): byte ranges split across the copy pool above 8 MiB.
static void gather_par(uint8_t *dst, const uint64_t *ptrs, const uint64_t *lens, const int64_t *offs,
                       uint64_t n_docs) {
    const uint64_t n = (uint64_t)offs[n_docs];
    auto range = [&](uint64_t lo, uint64_t hi) {  // copy bytes [lo, hi) of the packed batch
        uint64_t d = (uint64_t)(std::upper_bound(offs, offs + n_docs + 1, (int64_t)lo) - offs) - 1;
        for (; d < n_docs && (uint64_t)offs[d] < hi; ++d) {
            const uint64_t a = std::max<uint64_t>(lo, offs[d]), b = std::min<uint64_t>(hi, offs[d + 1]);
            if (a < b) memcpy(dst + a, reinterpret_cast<const uint8_t *>(ptrs[d]) + (a - offs[d]), b - a);
        }
    };
    const size_t per = 4u << 20;
    if (n <= 2 * per) {
        range(0, n);
        return;
    }
    CopyPool &pool = CopyPool::get();
    const unsigned parts = (unsigned)std::min<size_t>(pool.workers() + 1, (n + per - 1) / per);
    const uint64_t chunk = (n + parts - 1) / parts;
    pool.run(parts, [&](unsigned i) { range(std::min(n, i * chunk), std::min(n, (i + 1) * chunk)); });
}

static int ensure_pinned(gpubpe_ctx *ctx, size_t bytes) {
    if (ctx->pin_bytes >= bytes && ctx->pin) return GPUBPE_OK;
    if (ctx->pin) CK(cudaFreeHost(ctx->pin));
    ctx->pin = nullptr;
    ctx->pin_bytes = 0;
    const size_t nb = std::max<size_t>(bytes + bytes / 4, 1 << 20);
    CK(cudaHostAlloc(reinterpret_cast<void **>(&ctx->pin), nb, cudaHostAllocMapped));
    ++ctx->n_allocs;
    void *dev = nullptr;
    CK(cudaHostGetDevicePointer(&dev, ctx->pin, 0));
    ctx->pin_dev = static_cast<uint8_t *>(dev);
    ctx->pin_bytes = nb;
    return GPUBPE_OK;
}

static int ensure_host(gpubpe_ctx *ctx, uint8_t **p, uint8_t **p_dev, size_t *have, size_t bytes) {
    if (*have >= bytes && *p) return GPUBPE_OK;
    if (*p) CK(cudaFreeHost(*p));
    *p = nullptr;
    *have = 0;
    const size_t nb = std::max<size_t>(bytes + bytes / 8, 1 << 20);
    CK(cudaHostAlloc(reinterpret_cast<void **>(p), nb, p_dev ? cudaHostAllocMapped : 0));
    ++ctx->n_allocs;
    if (p_dev) {
        void *dev = nullptr;
        CK(cudaHostGetDevicePointer(&dev, *p, 0));
        *p_dev = static_cast<uint8_t *>(dev);
    }
    *have = nb;
    return GPUBPE_OK;
}

// Device alias of a pinned, device-mapped host pointer (gpubpe_host_alloc), else null.
static void *mapped_alias(const void *h) {
    cudaPointerAttributes pa{};
    void *d = nullptr;
    if (h && cudaPointerGetAttributes(&pa, h) == cudaSuccess && pa.type == cudaMemoryTypeHost)
        d = pa.devicePointer;
    cudaGetLastError();
    return d;
}

// gpubpe_encode_host for a large batch: parts of about `part_bytes` (whole
// documents; a larger document is a part of its own) run through a two-slot
// pipeline on three streams -- H2D of part i (s_copy), encode of part i-1
// (the caller's stream) and D2H of part i-2's ids (s_d2h) overlap; the encodes
// are enqueued back to back.  Documents are independent (chunker.py:139-179),
// so the parts' results concatenate.
//   input:  pinned caller bytes (gpubpe_host_alloc) are copied to the device
//           directly; pageable ones are staged through the slot's pinned buffer;
//   output: ids are DMA'd to a pinned caller buffer at their final position
//           (known once the previous part's id count is: the host reads each
//           part's offsets from mapped memory when it completes); a pageable
//           caller buffer receives them through the slot's pinned buffer.
// Overflow of the deferred-segment buffers is checked per part (drain) and
// the part re-encoded synchronously after growing them.
static int encode_host_streamed(gpubpe_ctx *ctx, const uint8_t *h_bytes, const int64_t *h_doc_offs,
                                uint64_t n_docs, uint64_t max_seq_len, uint64_t chunk_budget,
                                uint32_t *h_out_ids, int64_t *h_out_offs, uint64_t *n_ids_out,
                                float *kernel_ms, void *stream, uint64_t part_bytes) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!ctx->s_copy) CK(cudaStreamCreateWithFlags(&ctx->s_copy, cudaStreamNonBlocking));
    if (!ctx->s_d2h) CK(cudaStreamCreateWithFlags(&ctx->s_d2h, cudaStreamNonBlocking));
    if (!ctx->h_state_ss) {
        CK(cudaHostAlloc(reinterpret_cast<void **>(&ctx->h_state_ss), 2 * sizeof(EncodeState), 0));
        ++ctx->n_allocs;
    }
    for (auto &S : ctx->ss) {
        if (!S.ev_h2d) CK(cudaEventCreate(&S.ev_h2d));
        if (!S.ev_done) CK(cudaEventCreate(&S.ev_done));
        if (!S.ev_d2h) CK(cudaEventCreate(&S.ev_d2h));
    }
    const bool in_pinned = mapped_alias(h_bytes) != nullptr;
    const bool out_pinned = mapped_alias(h_out_ids) != nullptr;
    std::vector<std::pair<uint64_t, uint64_t>> parts;  // document ranges
    for (uint64_t d = 0; d < n_docs;) {
        uint64_t e = d + 1;
        while (e < n_docs && (uint64_t)(h_doc_offs[e + 1] - h_doc_offs[d]) <= part_bytes) ++e;
        parts.emplace_back(d, e);
        d = e;
    }
    const size_t P = parts.size();
    auto nb_of = [&](size_t i) { return (uint64_t)(h_doc_offs[parts[i].second] - h_doc_offs[parts[i].first]); };
    auto nd_of = [&](size_t i) { return parts[i].second - parts[i].first; };
    auto ids_off = [](uint64_t nd) { return ((nd + 1) * 8 + 255) & ~(size_t)255; };
    std::vector<uint64_t> base_of(P, 0), cnt_of(P, 0);
    EncodeState agg{};
    uint64_t base = 0, tiles = 0;
    const bool htime = getenv("GPUBPE_HOSTTIME") != nullptr;
    double t_wait = 0, t_out = 0, t_in = 0, t_enq = 0;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto us = [](auto x, auto y) { return std::chrono::duration<double, std::micro>(y - x).count(); };
    const auto t_start = now();
    auto encode_part = [&](size_t i) -> int {  // enqueue the encode of part i on s
        auto &S = ctx->ss[i & 1];
        const uint64_t nd = nd_of(i), nb = nb_of(i);
        uint8_t *din = static_cast<uint8_t *>(S.dev_in.p);
        const size_t o_offs = (nb + 255) & ~(size_t)255;
        int rc2 = gpubpe_encode(ctx, din, nb, reinterpret_cast<const int64_t *>(din + o_offs), nd, max_seq_len,
                                chunk_budget, static_cast<uint32_t *>(S.dev_out.p),
                                reinterpret_cast<int64_t *>(S.pin_out_dev), stream);
        if (rc2) return rc2;
        tiles += nb ? ctx->last_n_tiles : 0;
        const EncodeState *last = static_cast<const EncodeState *>(ctx->ws_state.p) + ((ctx->calls - 1) & 1);
        CK(cudaMemcpyAsync(&ctx->h_state_ss[i & 1], last, sizeof(EncodeState), cudaMemcpyDeviceToHost, s));
        CK(cudaEventRecord(S.ev_done, s));
        return GPUBPE_OK;
    };
    auto drain = [&](size_t i) -> int {  // part i encoded: offsets, counters, enqueue the D2H of its ids
        auto &S = ctx->ss[i & 1];
        auto t0 = now();
        CK(cudaEventSynchronize(S.ev_done));
        t_wait += us(t0, now());
        const uint64_t d = parts[i].first, nd = nd_of(i), nb = nb_of(i);
        if (nb && ctx->h_state_ss[i & 1].overflow) {
            // deferred-segment buffers overflowed: grow them, redo this part with the
            // synchronous check (its input is still in its slot)
            const EncodeState &o = ctx->h_state_ss[i & 1];
            int rc2;
            ctx->defer_check = false;
            tiles -= ctx->last_n_tiles;
            if ((rc2 = ensure(ctx, ctx->ws_recs, (o.bar >> 32) * sizeof(DefRec), false)) ||
                (rc2 = ensure(ctx, ctx->ws_arena, o.arena_used * 4, false)) || (rc2 = encode_part(i))) {
                ctx->defer_check = true;
                return rc2;
            }
            ctx->defer_check = true;
            CK(cudaStreamSynchronize(s));
        }
        const int64_t *lo = reinterpret_cast<const int64_t *>(S.pin_out);
        const uint64_t cnt = nb ? (uint64_t)lo[nd] : 0;
        if (cnt > nb)
            return fail(ctx, GPUBPE_ECUDA, "device produced %llu ids for %llu bytes", (unsigned long long)cnt,
                        (unsigned long long)nb);
        for (uint64_t j = 0; j <= nd; ++j) h_out_offs[d + j] = (int64_t)base + (nb ? lo[j] : 0);
        if (cnt) {
            void *to = out_pinned ? static_cast<void *>(h_out_ids + base) : static_cast<void *>(S.pin_out + ids_off(nd));
            CK(cudaMemcpyAsync(to, S.dev_out.p, cnt * 4, cudaMemcpyDeviceToHost, ctx->s_d2h));
        }
        CK(cudaEventRecord(S.ev_d2h, ctx->s_d2h));
        const EncodeState &st = ctx->h_state_ss[i & 1];
        if (nb) {
            agg.overflow |= st.overflow;
            agg.c.n_segments += st.c.n_segments;
            agg.c.memo_hits += st.c.memo_hits;
            agg.c.short_merges += st.c.short_merges;
            agg.c.medium_segments += st.c.medium_segments;
            agg.c.giant_segments += st.c.giant_segments;
            agg.c.giant_bytes += st.c.giant_bytes;
            agg.c.engine_passes += st.c.engine_passes;
        }
        base_of[i] = base;
        cnt_of[i] = cnt;
        base += cnt;
        return GPUBPE_OK;
    };
    auto complete = [&](size_t i) -> int {  // part i's ids are in the caller's buffer afterwards
        auto &S = ctx->ss[i & 1];
        auto t0 = now();
        CK(cudaEventSynchronize(S.ev_d2h));
        auto t1 = now();
        t_wait += us(t0, t1);
        if (!out_pinned && cnt_of[i]) copy_par(h_out_ids + base_of[i], S.pin_out + ids_off(nd_of(i)), cnt_of[i] * 4);
        t_out += us(t1, now());
        return GPUBPE_OK;
    };
    struct DeferGuard {  // overflow is checked per part in drain(), not per launch
        gpubpe_ctx *c;
        explicit DeferGuard(gpubpe_ctx *c_) : c(c_) { c->defer_check = true; }
        ~DeferGuard() { c->defer_check = false; }
    } guard(ctx);
    int rc;
    for (size_t i = 0; i < P; ++i) {
        auto &S = ctx->ss[i & 1];
        // slot i & 1 is free again once part i-2's ids left it (device side: the stream
        // wait below; a staged output also needs its host copy-out first)
        if (i >= 2 && !out_pinned && (rc = complete(i - 2))) return rc;
        const uint64_t d = parts[i].first, nd = nd_of(i), lo = (uint64_t)h_doc_offs[d], nb = nb_of(i);
        const size_t o_offs = (nb + 255) & ~(size_t)255, need_in = o_offs + (nd + 1) * 8;
        const size_t need_out = ids_off(nd) + (out_pinned ? 0 : std::max<uint64_t>(nb, 1) * 4);
        if ((rc = ensure_host(ctx, &S.pin_in, nullptr, &S.pin_in_bytes, in_pinned ? (nd + 1) * 8 : need_in)))
            return rc;
        if ((rc = ensure_host(ctx, &S.pin_out, &S.pin_out_dev, &S.pin_out_bytes, need_out))) return rc;
        if ((rc = ensure(ctx, S.dev_in, need_in, false))) return rc;
        if ((rc = ensure(ctx, S.dev_out, std::max<uint64_t>(nb, 1) * 4, false))) return rc;
        auto t0 = now();
        uint8_t *din = static_cast<uint8_t *>(S.dev_in.p);
        int64_t *po = reinterpret_cast<int64_t *>(in_pinned ? S.pin_in : S.pin_in + o_offs);
        for (uint64_t j = 0; j <= nd; ++j) po[j] = h_doc_offs[d + j] - (int64_t)lo;
        if (in_pinned) {
            if (nb) CK(cudaMemcpyAsync(din, h_bytes + lo, nb, cudaMemcpyHostToDevice, ctx->s_copy));
            CK(cudaMemcpyAsync(din + o_offs, po, (nd + 1) * 8, cudaMemcpyHostToDevice, ctx->s_copy));
        } else {
            copy_par(S.pin_in, h_bytes + lo, nb);
            CK(cudaMemcpyAsync(din, S.pin_in, need_in, cudaMemcpyHostToDevice, ctx->s_copy));
        }
        CK(cudaEventRecord(S.ev_h2d, ctx->s_copy));
        CK(cudaStreamWaitEvent(s, S.ev_h2d, 0));
        if (i >= 2) CK(cudaStreamWaitEvent(s, S.ev_d2h, 0));  // the slot's device ids went out
        auto t1 = now();
        t_in += us(t0, t1);
        if ((rc = encode_part(i))) return rc;
        t_enq += us(t1, now());
        if (i >= 1 && (rc = drain(i - 1))) return rc;
    }
    if (P && (rc = drain(P - 1))) return rc;
    if (out_pinned) {
        auto t0 = now();
        CK(cudaStreamSynchronize(ctx->s_d2h));
        t_wait += us(t0, now());
    } else {
        for (size_t i = P >= 2 ? P - 2 : 0; i < P; ++i)
            if ((rc = complete(i))) return rc;
    }
    if (htime)
        fprintf(stderr, "encode_host streamed: %zu parts (input %s, output %s), total %.0f us: stage+h2d %.0f | "
                "enqueue %.0f | wait %.0f | copy-out %.0f\n", P, in_pinned ? "pinned" : "staged",
                out_pinned ? "pinned" : "staged", us(t_start, now()), t_in, t_enq, t_wait, t_out);
    if (kernel_ms && P) CK(cudaEventElapsedTime(kernel_ms, ctx->ss[0].ev_h2d, ctx->ss[(P - 1) & 1].ev_d2h));
    agg.n_ids = base;
    *ctx->h_state = agg;
    ctx->state_fresh = true;
    ctx->last_n_bytes = (uint64_t)(h_doc_offs[n_docs] - h_doc_offs[0]);
    ctx->last_n_tiles = tiles;
    *n_ids_out = base;
    return GPUBPE_OK;
}


static int encode_host_core(gpubpe_ctx *ctx, const uint8_t *h_bytes, const StageFn *stage, uint64_t n_bytes,
                            const int64_t *h_doc_offs, uint64_t n_docs, uint64_t max_seq_len, uint64_t chunk_budget,
                            uint32_t *h_out_ids, int64_t *h_out_offs, uint64_t *n_ids_out, float *kernel_ms,
                            void *stream);

// The caller thread's current device is restored on return (the host entry
// points select the context's device themselves; callers need no device guard).
struct DeviceRestore {
    int prev = -1;
    DeviceRestore() { cudaGetDevice(&prev); }
    ~DeviceRestore() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

extern "C" __attribute__((visibility("default"))) int gpubpe_encode_host(
    gpubpe_ctx *ctx, const uint8_t *h_bytes, uint64_t n_bytes, const int64_t *h_doc_offs, uint64_t n_docs,
    uint64_t max_seq_len, uint64_t chunk_budget, uint32_t *h_out_ids, int64_t *h_out_offs,
    uint64_t *n_ids_out, float *kernel_ms, void *stream) {
    if (!ctx) return GPUBPE_EINVAL;
    DeviceRestore restore_device;
    if (!n_ids_out || (n_docs && (!h_doc_offs || !h_out_offs)) || (n_bytes && (!h_bytes || !h_out_ids)))
        return fail(ctx, GPUBPE_EINVAL, "null host pointer");
    return encode_host_core(ctx, h_bytes, nullptr, n_bytes, h_doc_offs, n_docs, max_seq_len, chunk_budget, h_out_ids,
                            h_out_offs, n_ids_out, kernel_ms, stream);
}

static int encode_host_core(gpubpe_ctx *ctx, const uint8_t *h_bytes, const StageFn *stage, uint64_t n_bytes,
                            const int64_t *h_doc_offs, uint64_t n_docs, uint64_t max_seq_len, uint64_t chunk_budget,
                            uint32_t *h_out_ids, int64_t *h_out_offs, uint64_t *n_ids_out, float *kernel_ms,
                            void *stream) {
    // wake the staging helpers now, so they are spinning when the pieces are ready
    struct StageCall {  // the helpers spin from here until the last piece is staged
        bool on;
        explicit StageCall(bool b) : on(b) {
            if (on) StagePool::get().begin();
        }
        void done() {
            if (on) StagePool::get().end();
            on = false;
        }
        ~StageCall() { done(); }
    } stage_call(n_bytes >= (128u << 10) && n_bytes <= (16u << 20) && !getenv("GPUBPE_NO_STAGE_POOL"));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    ctx->alloc_mark = ctx->n_allocs;
    struct HostCall {  // gpubpe_encode calls below keep this call's allocation mark
        gpubpe_ctx *c;
        explicit HostCall(gpubpe_ctx *c_) : c(c_) { c->host_call = true; }
        ~HostCall() { c->host_call = false; }
    } host_call_guard(ctx);
    CK(cudaSetDevice(ctx->device));
    *n_ids_out = 0;
    if (kernel_ms) *kernel_ms = 0.f;
    if (n_docs == 0) return GPUBPE_OK;
    {  // large batches stream through a two-slot pipeline (GPUBPE_STREAM_MB: part size, 0 = never)
        const char *env = getenv("GPUBPE_STREAM_MB");
        const long long part_mb = env ? atoll(env) : 32;
        const uint64_t part = (uint64_t)std::max(part_mb, 0ll) << 20;
        if (part && n_bytes > 2 * part && n_docs > 1 && !stage)
            return encode_host_streamed(ctx, h_bytes, h_doc_offs, n_docs, max_seq_len, chunk_budget, h_out_ids,
                                        h_out_offs, n_ids_out, kernel_ms, stream, part);
    }
    static const bool htime = getenv("GPUBPE_HOSTTIME") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto t_a = now();
    static const int env_mode = getenv("GPUBPE_HOSTMODE") ? atoi(getenv("GPUBPE_HOSTMODE")) : 3;
    const int mode = stage ? 3 : env_mode;  // gathered batches always stage through pinned pieces
    int rc;
    const size_t offs_b = (n_docs + 1) * 8;
    const size_t o_in = 0;
    const size_t o_doffs = (n_bytes + 255) & ~(size_t)255;
    const size_t o_ooffs = (o_doffs + offs_b + 255) & ~(size_t)255;
    const size_t o_ids = (o_ooffs + offs_b + 255) & ~(size_t)255;
    const size_t need = o_ids + std::max<uint64_t>(n_bytes, 1) * 4;
    if ((rc = ensure_pinned(ctx, need))) return rc;
    if (!ctx->io_ev[0])
        for (auto &e : ctx->io_ev) CK(cudaEventCreate(&e));
    if (!ctx->h_mirror) {
        CK(cudaHostAlloc(reinterpret_cast<void **>(&ctx->h_mirror), sizeof(StateMirror), cudaHostAllocMapped));
        CK(cudaHostGetDevicePointer(reinterpret_cast<void **>(&ctx->d_mirror), ctx->h_mirror, 0));
        ++ctx->n_allocs;
    }
    // the kernel's last CTA writes the results here (kernels.cu kernel_exit): no D2H copy
    volatile StateMirror *mir = ctx->h_mirror;
    mir->n_ids = ~0ull;  // (sentinel: a kernel that did not write falls back to a copy)
    const unsigned long long mtag = ++ctx->mirror_tag;
    ctx->cur_mirror = ctx->d_mirror;
    struct MirrorOff {
        gpubpe_ctx *c;
        ~MirrorOff() { c->cur_mirror = nullptr; }
    } mirror_off{ctx};
    uint8_t *pin = ctx->pin;
    uint8_t *dv = nullptr;  // device copy of the same layout (modes 0 and 2)
    if (mode != 1) {
        if ((rc = ensure(ctx, ctx->io_dev, need, false))) return rc;
        dv = static_cast<uint8_t *>(ctx->io_dev.p);
    }
    uint8_t *dout = mode == 3 ? ctx->pin_dev : dv;  // where the kernel writes ids and offsets (mode 3:
                                                    // mapped pinned memory, the stores overlap the kernel)
    // A caller buffer that is itself pinned and device-mapped (gpubpe_host_alloc)
    // receives the ids directly: no copy-out at all.
    uint32_t *d_ids_direct = (mode == 3 && n_bytes) ? static_cast<uint32_t *>(mapped_alias(h_out_ids)) : nullptr;
    // Large batches: the ids go to device memory and come back by one DMA once the
    // count is known (PCIe writes from the SMs drain at ~26 GB/s, the copy engine
    // moves ~55 GB/s; GPUBPE_DMA_IDS_MB, default 2: the crossover measured on C2)
    static const long long dma_mb = getenv("GPUBPE_DMA_IDS_MB") ? atoll(getenv("GPUBPE_DMA_IDS_MB")) : 2;
    const bool dma_ids = mode == 3 && dma_mb >= 0 && n_bytes >= ((uint64_t)dma_mb << 20) && n_bytes;
    uint32_t *k_ids = dma_ids ? reinterpret_cast<uint32_t *>(dv + o_ids)
                              : d_ids_direct ? d_ids_direct : reinterpret_cast<uint32_t *>(dout + o_ids);
    // overlapped launch (one pageable buffer of 128 KiB .. 16 MiB, default mode):
    // ~4 pieces, the kernel enqueued before them
    const bool no_overlap = getenv("GPUBPE_NO_OVERLAP") != nullptr;  // (per call: tests switch it)
    // (every H2D copy costs ~7 us of setup on this PCIe 5 link, measured by
    // tools/overlap_probe.cu: one piece unless GPUBPE_OV_PIECES says otherwise)
    // (gathered batches: GPUBPE_OV_GATHER pieces, default 4 -- their staging is the long part)
    static const int ov_pieces = getenv("GPUBPE_OV_PIECES") ? std::max(1, atoi(getenv("GPUBPE_OV_PIECES"))) : 1;
    static const int ov_gather = getenv("GPUBPE_OV_GATHER") ? atoi(getenv("GPUBPE_OV_GATHER")) : 4;
    const int pieces = stage ? std::max(1, ov_gather) : ov_pieces;
    const size_t ov_piece = std::max<size_t>(32u << 10, ((n_bytes / pieces) + 4095) & ~(size_t)4095);
    const bool overlap = !no_overlap && mode == 3 && (!stage || ov_gather > 0) && ctx->mode == GPUBPE_MODE_DEFAULT &&
                         n_bytes >= (128u << 10) && n_bytes <= (16u << 20) &&
                         (n_bytes + ov_piece - 1) / ov_piece <= (size_t)ARRIVE_MAX && (stage || !mapped_alias(h_bytes));
    if (mode == 1) {  // zero-copy: the kernel reads and writes mapped host memory
        copy_par(pin + o_in, h_bytes, n_bytes);
        memcpy(pin + o_doffs, h_doc_offs, offs_b);
        dv = ctx->pin_dev;
    } else if (mode == 2) {  // pageable copies straight from the caller's buffers
        CK(cudaMemcpyAsync(dv + o_doffs, h_doc_offs, offs_b, cudaMemcpyHostToDevice, s));
        if (n_bytes) CK(cudaMemcpyAsync(dv + o_in, h_bytes, n_bytes, cudaMemcpyHostToDevice, s));
    } else if (overlap) {
        // overlapped: the input (one piece: every H2D copy costs ~7 us of setup
        // here) is staged by the helpers and DMA'd on s_copy, followed by its
        // arrival word; the kernel is enqueued right after on the caller's
        // stream, so its launch and prologue run while the DMA is in flight and
        // its tiles wait for the word.  The document offsets go first.
        if (!ctx->d_arrive) {
            CK(cudaMalloc(&ctx->d_arrive, ARRIVE_MAX * ARRIVE_STRIDE * sizeof(unsigned int)));
            CK(cudaMemset(ctx->d_arrive, 0, ARRIVE_MAX * ARRIVE_STRIDE * sizeof(unsigned int)));
            CK(cudaHostAlloc(reinterpret_cast<void **>(&ctx->h_tag), 64, 0));
            ctx->n_allocs += 2;
        }
        if (!ctx->s_copy) CK(cudaStreamCreateWithFlags(&ctx->s_copy, cudaStreamNonBlocking));
        if (++ctx->arrive_tag == 0) ctx->arrive_tag = 1;  // (words start at 0)
        *ctx->h_tag = ctx->arrive_tag;
        memcpy(pin + o_doffs, h_doc_offs, offs_b);
        CK(cudaMemcpyAsync(dv + o_doffs, pin + o_doffs, offs_b, cudaMemcpyHostToDevice, ctx->s_copy));
        const unsigned n_pieces = (unsigned)((n_bytes + ov_piece - 1) / ov_piece);
        static const bool ovt = getenv("GPUBPE_HOSTTIME") && atoi(getenv("GPUBPE_HOSTTIME")) == 3;
        static cudaEvent_t oev[3];
        if (ovt && !oev[0])
            for (auto &e : oev) cudaEventCreate(&e);
        auto th0 = now();
        if (ovt) cudaEventRecord(oev[0], ctx->s_copy);
        decltype(th0) th1 = th0;
        for (unsigned k = 0; k < n_pieces; ++k) {
            const size_t lo = (size_t)k * ov_piece, len = std::min<size_t>(ov_piece, n_bytes - lo);
            if (stage) StagePool::get().gather(pin + o_in + lo, *stage, lo, lo + len);
            else StagePool::get().copy(pin + o_in + lo, h_bytes + lo, len);
            if (k == 0) th1 = now();
            CK(cudaMemcpyAsync(dv + o_in + lo, pin + o_in + lo, len, cudaMemcpyHostToDevice, ctx->s_copy));
            CK(cudaMemcpyAsync(ctx->d_arrive + ARRIVE_STRIDE * k, ctx->h_tag, sizeof(unsigned int),
                               cudaMemcpyHostToDevice, ctx->s_copy));
        }
        if (ovt) cudaEventRecord(oev[1], ctx->s_copy);
        auto th2 = now();
        CK(cudaEventRecord(ctx->io_ev[0], s));
        ctx->cur_arrive = ctx->d_arrive;
        ctx->cur_piece = ov_piece;
        const bool dc = ctx->defer_check;
        ctx->defer_check = true;  // the overflow check waits for the final synchronisation
        rc = gpubpe_encode(ctx, dv + o_in, n_bytes, reinterpret_cast<const int64_t *>(dv + o_doffs), n_docs,
                           max_seq_len, chunk_budget,
                           k_ids,
                           reinterpret_cast<int64_t *>(dout + o_ooffs), stream);
        ctx->defer_check = dc;
        ctx->cur_arrive = nullptr;
        ctx->cur_piece = 0;
        if (rc) return rc;
        if (ovt) {  // GPUBPE_HOSTTIME=3: host and device timeline of the overlapped call
            cudaEventRecord(oev[2], s);
            auto th3 = now();
            cudaStreamSynchronize(s);
            auto th4 = now();
            float dma, ker;
            cudaEventElapsedTime(&dma, oev[0], oev[1]);
            cudaEventElapsedTime(&ker, oev[0], oev[2]);
            auto us = [](auto x, auto y) { return std::chrono::duration<double, std::micro>(y - x).count(); };
            fprintf(stderr, "overlap: host entry->stage start %.1f | staged %.1f | DMAs enqueued %.1f | launched %.1f | "
                            "synced %.1f us; GPU from the first DMA: data in %.1f | kernel end %.1f us\n",
                    us(t_a, th0), us(t_a, th1), us(t_a, th2), us(t_a, th3), us(t_a, th4), dma * 1e3, ker * 1e3);
        }
    } else if (n_bytes && !stage && mapped_alias(h_bytes)) {  // caller bytes already pinned: no staging copy
        memcpy(pin + o_doffs, h_doc_offs, offs_b);
        CK(cudaMemcpyAsync(dv + o_in, h_bytes, n_bytes, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(dv + o_doffs, pin + o_doffs, offs_b, cudaMemcpyHostToDevice, s));
    } else {  // pinned staging in 4 MiB pieces; staging of piece k+1 overlaps the DMA of piece k;
              // the doc offsets ride with the last piece (they follow the bytes in the layout)
        memcpy(pin + o_doffs, h_doc_offs, offs_b);
        // ~4 pieces (64 KiB .. 4 MiB) so the DMA starts after the first one is staged
        const char *pe = getenv("GPUBPE_PIECE_KB");
        const size_t piece = pe ? std::max<size_t>(4096, (size_t)atoll(pe) << 10)
                                : std::min<size_t>(4u << 20, std::max<size_t>(64u << 10, ((n_bytes / 4) + 65535) & ~(size_t)65535));
        // pieces of 128 KiB .. 4 MiB: split across the staging helpers
        const bool helpers = piece >= (128u << 10) && piece <= (4u << 20) && !getenv("GPUBPE_NO_STAGE_POOL");
        auto copy_piece = [&](uint8_t *dst, const uint8_t *src, size_t len) {
            if (helpers) StagePool::get().copy(dst, src, len);
            else copy_par(dst, src, len);
        };
        size_t lo = 0;
        static const bool tl = getenv("GPUBPE_HOSTTIME") && atoi(getenv("GPUBPE_HOSTTIME")) == 2;
        static cudaEvent_t tev[10];
        int ntev = 0;
        if (tl && !tev[0])
            for (auto &e : tev) cudaEventCreate(&e);
        if (tl) cudaEventRecord(tev[ntev++], s);
        auto stage_piece = [&](uint8_t *dst, uint64_t a, uint64_t b) {
            if (helpers) StagePool::get().gather(dst, *stage, a, b);
            else (*stage)(dst, a, b);
        };
        for (; lo + piece < n_bytes; lo += piece) {
            if (stage) stage_piece(pin + o_in + lo, lo, lo + piece);
            else copy_piece(pin + o_in + lo, h_bytes + lo, piece);
            CK(cudaMemcpyAsync(dv + o_in + lo, pin + o_in + lo, piece, cudaMemcpyHostToDevice, s));
            if (tl && ntev < 8) cudaEventRecord(tev[ntev++], s);
        }
        if (stage) stage_piece(pin + o_in + lo, lo, n_bytes);
        else copy_piece(pin + o_in + lo, h_bytes + lo, n_bytes - lo);
        CK(cudaMemcpyAsync(dv + o_in + lo, pin + o_in + lo, o_doffs + offs_b - lo, cudaMemcpyHostToDevice, s));
        if (tl) {  // GPU timeline of the pieces (GPUBPE_HOSTTIME=2): printed after the kernel
            cudaEventRecord(tev[ntev++], s);
            ctx->tl_n = ntev;
            ctx->tl_ev = tev;
        }
    }
    stage_call.done();
    auto t_b = now();
    if (!overlap) {
        CK(cudaEventRecord(ctx->io_ev[0], s));
        rc = gpubpe_encode(ctx, dv + o_in, n_bytes, reinterpret_cast<const int64_t *>(dv + o_doffs), n_docs,
                           max_seq_len, chunk_budget,
                           k_ids,
                           reinterpret_cast<int64_t *>(dout + o_ooffs), stream);
        if (rc) return rc;
    }
    CK(cudaEventRecord(ctx->io_ev[1], s));
    if (mode != 1 && mode != 3) CK(cudaMemcpyAsync(pin + o_ooffs, dv + o_ooffs, offs_b, cudaMemcpyDeviceToHost, s));
    auto t_c = now();
    // Wait for the results: with mapped outputs (mode 3) the kernel's last CTA
    // writes the mirror after every store is visible to the host (system-scope
    // fences), ~10 us before a stream synchronisation would return; the stream
    // is polled now and then so a failed or mirror-less launch still ends the wait.
    bool synced = false;
    if (mode == 3 && n_bytes) {
        for (unsigned it = 1;; ++it) {
            if (mir->done == mtag) break;
            if ((it & 1023) == 0) {
                const cudaError_t q = cudaStreamQuery(s);
                if (q == cudaSuccess) break;
                if (q != cudaErrorNotReady) CK(q);
            }
            cpu_relax();
        }
    }
    if (!(mode == 3 && n_bytes && mir->done == mtag && !mir->overflow)) {
        CK(cudaStreamSynchronize(s));
        synced = true;
    }
    auto t_d = now();
    ctx->cur_mirror = nullptr;
    if (n_bytes) {  // the counters, from the mirror (or, if the kernel did not fill it, a copy)
        if (mir->n_ids != ~0ull) {
            ctx->h_state->n_ids = mir->n_ids;
            ctx->h_state->overflow = mir->overflow;
            ctx->h_state->c = *const_cast<const PassCounters *>(&mir->c);
        } else {
            const EncodeState *last = static_cast<const EncodeState *>(ctx->ws_state.p) + ((ctx->calls - 1) & 1);
            CK(cudaMemcpy(ctx->h_state, last, sizeof(EncodeState), cudaMemcpyDeviceToHost));
        }
    }
    if (ctx->tl_n) {
        float ms;
        fprintf(stderr, "timeline (us from the first piece's enqueue):");
        for (int k = 1; k < ctx->tl_n; ++k) {
            cudaEventElapsedTime(&ms, ctx->tl_ev[0], ctx->tl_ev[k]);
            fprintf(stderr, " piece%d %.1f", k - 1, ms * 1e3);
        }
        cudaEventElapsedTime(&ms, ctx->tl_ev[0], ctx->io_ev[0]);
        fprintf(stderr, " | kernel enqueued-point %.1f", ms * 1e3);
        cudaEventElapsedTime(&ms, ctx->tl_ev[0], ctx->io_ev[1]);
        fprintf(stderr, " | kernel end %.1f\n", ms * 1e3);
        ctx->tl_n = 0;
    }
    ctx->state_fresh = n_bytes != 0;
    if (overlap && ctx->dbg_buf && getenv("GPUBPE_DEBUG")) dump_debug(ctx, s);
    if (overlap && ctx->h_state->overflow) {
        // deferred-segment buffers too small (checked here, not at the launch):
        // the input is on the device now; re-run the plain path, which grows them
        rc = gpubpe_encode(ctx, dv + o_in, n_bytes, reinterpret_cast<const int64_t *>(dv + o_doffs), n_docs,
                           max_seq_len, chunk_budget,
                           k_ids,
                           reinterpret_cast<int64_t *>(dout + o_ooffs), stream);
        if (rc) return rc;
        const EncodeState *last = static_cast<const EncodeState *>(ctx->ws_state.p) + ((ctx->calls - 1) & 1);
        CK(cudaMemcpyAsync(ctx->h_state, last, sizeof(EncodeState), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    const int64_t *p_oo = reinterpret_cast<const int64_t *>(pin + o_ooffs);
    const uint64_t total = n_bytes ? (uint64_t)p_oo[n_docs] : 0;
    if (total > n_bytes)
        return fail(ctx, GPUBPE_ECUDA, "device produced %llu ids for %llu bytes", (unsigned long long)total,
                    (unsigned long long)n_bytes);
    memcpy(h_out_offs, p_oo, offs_b);
    if (total) {
        if (dma_ids) {  // one D2H copy of exactly the ids produced
            CK(cudaMemcpyAsync(d_ids_direct ? static_cast<void *>(h_out_ids) : static_cast<void *>(pin + o_ids),
                               dv + o_ids, total * 4, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            if (!d_ids_direct) copy_par(h_out_ids, pin + o_ids, total * 4);
        } else if (d_ids_direct) {
            // already in place
        } else if (mode == 1 || mode == 3) {
            copy_par(h_out_ids, pin + o_ids, total * 4);
        } else if (mode == 2) {
            CK(cudaMemcpy(h_out_ids, dv + o_ids, total * 4, cudaMemcpyDeviceToHost));
        } else {
            CK(cudaMemcpyAsync(pin + o_ids, dv + o_ids, total * 4, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            copy_par(h_out_ids, pin + o_ids, total * 4);
        }
    }
    if (kernel_ms) {  // from the events once complete; else the host's view (enqueue to results)
        if (synced || cudaEventQuery(ctx->io_ev[1]) == cudaSuccess)
            CK(cudaEventElapsedTime(kernel_ms, ctx->io_ev[0], ctx->io_ev[1]));
        else
            *kernel_ms = (float)(std::chrono::duration<double, std::milli>(t_d - t_b).count());
        cudaGetLastError();
    }
    *n_ids_out = total;
    if (htime) {
        auto t_e = now();
        auto us = [](auto x, auto y) { return std::chrono::duration<double, std::micro>(y - x).count(); };
        fprintf(stderr, "encode_host: stage+h2d enqueue %.1f | encode enqueue %.1f | sync wait %.1f | copy-out %.1f us\n",
                us(t_a, t_b), us(t_b, t_c), us(t_c, t_d), us(t_d, t_e));
    }
    return GPUBPE_OK;
}

extern "C" __attribute__((visibility("default"))) int gpubpe_encode_host_gather(
    gpubpe_ctx *ctx, const uint64_t *h_ptrs, const uint64_t *h_lens, uint64_t n_docs, uint64_t max_seq_len,
    uint64_t chunk_budget, uint32_t *h_out_ids, int64_t *h_out_offs, uint64_t *n_ids_out, float *kernel_ms,
    void *stream) {
    if (!ctx) return GPUBPE_EINVAL;
    if (!n_ids_out || (n_docs && (!h_ptrs || !h_lens || !h_out_offs)))
        return fail(ctx, GPUBPE_EINVAL, "null host pointer");
    std::vector<int64_t> offs(n_docs + 1, 0);
    for (uint64_t d = 0; d < n_docs; ++d) {
        if (h_lens[d] && !h_ptrs[d]) return fail(ctx, GPUBPE_EINVAL, "document %llu: null pointer", (unsigned long long)d);
        offs[d + 1] = offs[d] + (int64_t)h_lens[d];
    }
    const uint64_t n = (uint64_t)offs[n_docs];
    const char *env = getenv("GPUBPE_STREAM_MB");
    const uint64_t part = (uint64_t)std::max(env ? atoll(env) : 32ll, 0ll) << 20;
    if (n == 0 || (part && n > 2 * part && n_docs > 1)) {  // (large batches: contiguous copy, then streamed)
        std::vector<uint8_t> buf(std::max<uint64_t>(n, 1));
        gather_par(buf.data(), h_ptrs, h_lens, offs.data(), n_docs);
        return gpubpe_encode_host(ctx, buf.data(), n, offs.data(), n_docs, max_seq_len, chunk_budget, h_out_ids,
                                  h_out_offs, n_ids_out, kernel_ms, stream);
    }
    // stage the pieces straight from the documents into pinned memory (each piece
    // DMA'd while the next one is gathered): one host copy, no join
    const StageFn stage = [&](uint8_t *dst, uint64_t lo, uint64_t hi) {
        uint64_t d = (uint64_t)(std::upper_bound(offs.begin(), offs.end(), (int64_t)lo) - offs.begin()) - 1;
        for (; d < n_docs && (uint64_t)offs[d] < hi; ++d) {
            const uint64_t a = std::max<uint64_t>(lo, offs[d]), b = std::min<uint64_t>(hi, offs[d + 1]);
            if (a < b) memcpy(dst + (a - lo), reinterpret_cast<const uint8_t *>(h_ptrs[d]) + (a - offs[d]), b - a);
        }
    };
    if (!h_out_ids) return fail(ctx, GPUBPE_EINVAL, "null host pointer");
    return encode_host_core(ctx, nullptr, &stage, n, offs.data(), n_docs, max_seq_len, chunk_budget, h_out_ids,
                            h_out_offs, n_ids_out, kernel_ms, stream);
}

extern "C" __attribute__((visibility("default"))) int gpubpe_host_alloc(int device, uint64_t bytes, void **out) {
    if (!out) return GPUBPE_EINVAL;
    *out = nullptr;
    if (cudaSetDevice(device) != cudaSuccess) return GPUBPE_ECUDA;
    void *p = nullptr;
    const cudaError_t e = cudaHostAlloc(&p, std::max<uint64_t>(bytes, 1), cudaHostAllocMapped | cudaHostAllocPortable);
    if (e != cudaSuccess) return e == cudaErrorMemoryAllocation ? GPUBPE_ENOMEM : GPUBPE_ECUDA;
    *out = p;
    return GPUBPE_OK;
}

extern "C" __attribute__((visibility("default"))) void gpubpe_host_free(void *p) {
    if (p) cudaFreeHost(p);
}

extern "C" __attribute__((visibility("default"))) int gpubpe_query(gpubpe_ctx *ctx, void *stream, gpubpe_stats *out) {
    if (!ctx || !out) return GPUBPE_EINVAL;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    memset(out, 0, sizeof *out);
    if (ctx->state_fresh) {
        // gpubpe_encode_host already brought the last encode's state back
    } else if (ctx->ws_state.p && ctx->calls) {
        const EncodeState *last = static_cast<const EncodeState *>(ctx->ws_state.p) + ((ctx->calls - 1) & 1);
        CK(cudaMemcpyAsync(ctx->h_state, last, sizeof(EncodeState), cudaMemcpyDeviceToHost, s));
    } else {
        memset(ctx->h_state, 0, sizeof(EncodeState));
    }
    if (!ctx->state_fresh) CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
    const EncodeState &st = *ctx->h_state;
    if (st.overflow) return fail(ctx, GPUBPE_ECUDA, "device reported an unrecovered buffer overflow");
    out->n_bytes = ctx->last_n_bytes;
    out->n_ids = st.n_ids;
    out->passes = out->n_bytes - st.n_ids;
    out->n_segments = st.c.n_segments;
    out->memo_hits = st.c.memo_hits;
    out->short_merges = st.c.short_merges;
    out->medium_segments = st.c.medium_segments;
    out->giant_segments = st.c.giant_segments;
    out->giant_bytes = st.c.giant_bytes;
    out->engine_passes = st.c.engine_passes;
    out->tiles = ctx->last_n_bytes ? ctx->last_n_tiles : 0;
    out->overflow = st.overflow;
    out->well_formed = (uint64_t)ctx->T.well_formed;
    out->allocations = ctx->n_allocs - ctx->alloc_mark;
    return GPUBPE_OK;
}

extern "C" __attribute__((visibility("default"))) int gpubpe_set_vocab(gpubpe_ctx *ctx, const uint32_t *ids,
                                                                         const uint8_t *bytes,
                                                                         const uint64_t *offs, uint64_t n) {
    if (!ctx || (n && (!ids || !bytes || !offs))) return GPUBPE_EINVAL;
    CK(cudaSetDevice(ctx->device));
    uint64_t max_id = 0;
    for (uint64_t i = 0; i < n; ++i) max_id = std::max<uint64_t>(max_id, ids[i]);
    if (n && max_id >= (1ull << 26)) return fail(ctx, GPUBPE_EINVAL, "decode: ids must be < 2^26");
    // strings 16-B aligned and zero-padded: the kernel fetches them with 16-B loads;
    // vinfo = (offset / 16) << 8 | min(length, LEN_EXT); every length (empty symbols
    // and strings of any size included, decode_tokens semantics) in vlong
    std::vector<uint32_t> vinfo(n ? max_id + 1 : 1, GPUBPE_INF), vlong(vinfo.size(), 0);
    std::vector<uint8_t> blob;
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t len = offs[i + 1] - offs[i];
        if (len >= (1ull << 31)) return fail(ctx, GPUBPE_EINVAL, "decode: a vocab string exceeds 2 GiB");
        const uint64_t at = blob.size();
        if ((at >> 4) >= (1ull << 24)) return fail(ctx, GPUBPE_EINVAL, "decode: vocab strings exceed 256 MiB");
        blob.insert(blob.end(), bytes + offs[i], bytes + offs[i + 1]);
        blob.resize((blob.size() + 15) & ~(size_t)15, 0);
        vinfo[ids[i]] = (uint32_t)((at >> 4) << 8) | (uint32_t)std::min<uint64_t>(len, LEN_EXT);
        vlong[ids[i]] = (uint32_t)len;
    }
    blob.resize(blob.size() + 16, 0);
    const uint64_t blob_b = blob.size();
    // per id: a 16-B record (length byte, then the string if it fits, else its
    // blob chunk and length) and a 1-byte length table (the two-pass decode's
    // first pass; LEN_EXT for empty and >= 255-byte strings, 0 for unknown ids)
    // (vrec has one zero record more, at index n_vocab: unknown ids clamp to it)
    std::vector<uint8_t> vrec((vinfo.size() + 1) * 16, 0), vlen(vinfo.size(), 0);
    bool ext = false;
    for (size_t i = 0; i < vinfo.size(); ++i) {
        if (vinfo[i] == GPUBPE_INF) continue;
        const uint32_t len = vlong[i], chunk = vinfo[i] >> 8;
        uint8_t *r = &vrec[16 * i];
        r[0] = (uint8_t)std::min<uint32_t>(len, LEN_EXT);
        if (len <= 15) {
            memcpy(r + 1, &blob[16ull * chunk], len);
        } else {
            memcpy(r + 4, &chunk, 4);
            memcpy(r + 8, &len, 4);
        }
        vlen[i] = (uint8_t)(len == 0 || len >= LEN_EXT ? LEN_EXT : len);
        ext = ext || vlen[i] == LEN_EXT;
    }
    ctx->vocab_ext = ext;
    if (ctx->d_vrec) cudaFree(ctx->d_vrec);
    if (ctx->d_vlen) cudaFree(ctx->d_vlen);
    ctx->d_vrec = nullptr;
    ctx->d_vlen = nullptr;
    CK(cudaMalloc(&ctx->d_vrec, vrec.size()));
    CK(cudaMemcpy(ctx->d_vrec, vrec.data(), vrec.size(), cudaMemcpyHostToDevice));
    CK(cudaMalloc(&ctx->d_vlen, vlen.size()));
    CK(cudaMemcpy(ctx->d_vlen, vlen.data(), vlen.size(), cudaMemcpyHostToDevice));
    if (ctx->d_vlong) cudaFree(ctx->d_vlong);
    ctx->d_vlong = nullptr;
    CK(cudaMalloc(&ctx->d_vlong, vlong.size() * 4));
    CK(cudaMemcpy(ctx->d_vlong, vlong.data(), vlong.size() * 4, cudaMemcpyHostToDevice));
    if (ctx->d_vinfo) cudaFree(ctx->d_vinfo);
    if (ctx->d_vblob) cudaFree(ctx->d_vblob);
    ctx->d_vinfo = nullptr;
    ctx->d_vblob = nullptr;
    CK(cudaMalloc(&ctx->d_vinfo, vinfo.size() * 4));
    CK(cudaMemcpy(ctx->d_vinfo, vinfo.data(), vinfo.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&ctx->d_vblob, blob_b));
    CK(cudaMemcpy(ctx->d_vblob, blob.data(), blob_b, cudaMemcpyHostToDevice));
    ctx->n_vocab_dec = (uint32_t)vinfo.size();
    CK(setup_decode());
    int blocks = 0;
    CK(decode_occupancy(&blocks));
    ctx->dec_grid = ctx->num_sms * std::max(1, blocks);
    CK(decode_rows_occupancy(&blocks));
    ctx->dec_rows_grid = ctx->num_sms * std::max(1, blocks);
    return GPUBPE_OK;
}

extern "C" __attribute__((visibility("default"))) int gpubpe_decode(gpubpe_ctx *ctx, const uint32_t *d_ids, uint64_t n_ids,
                                                                      const int64_t *d_id_offs, uint64_t n_seqs,
                                                                      uint8_t *d_out, uint64_t out_cap,
                                                                      int64_t *d_out_offs, uint64_t *n_bytes_out,
                                                                      uint64_t *bad_index, void *stream) {
    if (!ctx || !n_bytes_out || !bad_index) return GPUBPE_EINVAL;
    *n_bytes_out = 0;
    *bad_index = ~0ull;  // set before any argument check: EINVAL with an index means an unknown id
    if (!ctx->d_vinfo) return fail(ctx, GPUBPE_EINVAL, "decode: no vocabulary (gpubpe_set_vocab)");
    if (n_seqs && (!d_id_offs || !d_out_offs)) return fail(ctx, GPUBPE_EINVAL, "decode: null offsets");
    // the kernels store bytes in 16-byte vectors (decode.cu); ids may sit at any 4-byte offset
    if ((reinterpret_cast<uintptr_t>(d_out) & 15) || (reinterpret_cast<uintptr_t>(d_ids) & 3))
        return fail(ctx, GPUBPE_EINVAL, "decode: d_out must be 16-byte aligned and d_ids 4-byte aligned");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CK(cudaSetDevice(ctx->device));
    *n_bytes_out = 0;
    *bad_index = ~0ull;
    if (n_ids == 0) {
        if (n_seqs) CK(cudaMemsetAsync(d_out_offs, 0, (n_seqs + 1) * 8, s));
        return GPUBPE_OK;
    }
    const uint64_t n_tiles = (n_ids + decode_tile_ids() - 1) / decode_tile_ids();
    int rc;
    if ((rc = ensure(ctx, ctx->dec_state, sizeof(DecodeState), false))) return rc;
    if (ctx->dec_status.bytes < n_tiles * 8) ctx->dec_epoch = 0;
    if ((rc = ensure(ctx, ctx->dec_status, n_tiles * 8, true))) return rc;
    if (++ctx->dec_epoch >= (1u << 20)) {
        CK(cudaMemsetAsync(ctx->dec_status.p, 0, ctx->dec_status.bytes, s));
        ctx->dec_epoch = 1;
    }
    // the state goes down and comes back through the pinned state buffer (a pageable
    // source would make the first copy a staged, host-blocking one)
    static_assert(sizeof(EncodeState) >= 2 * sizeof(DecodeState), "pinned state buffer too small");
    DecodeState *hs = reinterpret_cast<DecodeState *>(ctx->h_state);
    ctx->state_fresh = false;
    hs[0] = DecodeState{0, 0, 0, ~0ull};
    DecodeState *d_st = static_cast<DecodeState *>(ctx->dec_state.p);
    CK(cudaMemcpyAsync(d_st, &hs[0], sizeof(DecodeState), cudaMemcpyHostToDevice, s));
    DecodeParams P{};
    P.vinfo = ctx->d_vinfo;
    P.blob = ctx->d_vblob;
    P.vrec = ctx->d_vrec;
    P.vlen = ctx->d_vlen;
    P.vlong = ctx->d_vlong;
    P.ext = ctx->vocab_ext ? 1u : 0u;
    P.n_vocab = ctx->n_vocab_dec;
    P.ids = d_ids;
    P.n_ids = n_ids;
    P.id_offs = reinterpret_cast<const long long *>(d_id_offs);
    P.n_seqs = n_seqs;
    P.out = d_out;
    P.out_cap = out_cap;
    P.out_offs = reinterpret_cast<long long *>(d_out_offs);
    P.st = d_st;
    P.status = static_cast<unsigned long long *>(ctx->dec_status.p);
    P.n_tiles = n_tiles;
    P.epoch = ctx->dec_epoch;
    P.aligned = (reinterpret_cast<uintptr_t>(d_ids) & 15) == 0;
    P.tile_base = nullptr;
    const char *tp_env = getenv("GPUBPE_DEC_TWOPASS_MIN");  // tiles (tuning)
    // two passes (tile totals + scan, then the warp-per-row kernel) from ~1.25 tiles per
    // CTA of the one-pass kernel: measured crossover between 1 M ids (256 tiles: one pass
    // 46 us, two 54 us) and 2.1 M ids (515 tiles: 62 vs 57 us)
    const uint64_t tp_min = tp_env ? strtoull(tp_env, nullptr, 10) : (5 * (uint64_t)ctx->dec_grid) / 4;
    if (n_tiles >= tp_min && !getenv("GPUBPE_DEC_LOOKBACK")) {
        if ((rc = ensure(ctx, ctx->dec_tiles, n_tiles * 16 + n_tiles * 4 * (decode_tile_ids() / 128), false)))
            return rc;
        unsigned long long *tb = static_cast<unsigned long long *>(ctx->dec_tiles.p);
        const bool rows = !getenv("GPUBPE_DEC_TILES");
        P.row_bytes = rows ? reinterpret_cast<uint32_t *>(tb + 2 * n_tiles) : nullptr;
        CK(launch_decode_offsets(P, tb, tb + n_tiles, s));
        P.tile_base = tb + n_tiles;
        if (rows) CK(launch_decode_rows(P, ctx->dec_rows_grid, s));
        else CK(launch_decode(P, (int)std::min<uint64_t>(n_tiles, (uint64_t)ctx->dec_grid), s));
    } else {
        CK(launch_decode(P, (int)std::min<uint64_t>(n_tiles, (uint64_t)ctx->dec_grid), s));
    }
    DecodeState h;
    CK(cudaMemcpyAsync(&hs[1], d_st, sizeof h, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    memcpy(&h, &hs[1], sizeof h);
    ctx->state_fresh = false;
    if (h.bad != ~0ull) {
        *bad_index = h.bad;
        return fail(ctx, GPUBPE_EINVAL, "id at index %llu not in vocabulary", (unsigned long long)h.bad);
    }
    if (h.need) {
        *n_bytes_out = h.need;
        return fail(ctx, GPUBPE_ERANGE, "decode output needs %llu bytes (capacity %llu)",
                    (unsigned long long)h.need, (unsigned long long)out_cap);
    }
    *n_bytes_out = h.n_bytes;
    return GPUBPE_OK;
}

extern "C" __attribute__((visibility("default"))) int gpubpe_set_pretok(gpubpe_ctx *ctx, const uint8_t *classes,
                                                                          uint64_t n_cps) {
    if (!ctx || !classes || n_cps < 128 || n_cps > 0x110000) return GPUBPE_EINVAL;
    CK(cudaSetDevice(ctx->device));
    if (ctx->d_pt_classes) cudaFree(ctx->d_pt_classes);
    ctx->d_pt_classes = nullptr;
    const size_t nb = (n_cps + 3) / 4;
    CK(cudaMalloc(&ctx->d_pt_classes, nb));
    CK(cudaMemcpy(ctx->d_pt_classes, classes, nb, cudaMemcpyHostToDevice));
    for (int c = 0; c < 128; ++c) ctx->pt_ascii[c] = (classes[c >> 2] >> (2 * (c & 3))) & 3;
    ctx->pt_n_cps = (uint32_t)n_cps;
    return GPUBPE_OK;
}

extern "C" __attribute__((visibility("default"))) int gpubpe_set_mode(gpubpe_ctx *ctx, uint32_t mode) {
    if (!ctx || mode > GPUBPE_MODE_GPT2_REGEX) return GPUBPE_EINVAL;
    if (mode == GPUBPE_MODE_GPT2_REGEX && !ctx->d_pt_classes)
        return fail(ctx, GPUBPE_EINVAL, "GPT-2 regex mode needs gpubpe_set_pretok first");
    ctx->mode = mode;
    return GPUBPE_OK;
}

static int merge_tokens(gpubpe_ctx *ctx, const uint32_t *d_tokens, const uint64_t *h_offs, uint64_t n_seqs,
                        uint32_t *d_out, uint64_t *h_counts, uint64_t *d_trace, int64_t fault_seq, void *stream) {
    if (!ctx || (n_seqs && (!h_offs || !h_counts))) return GPUBPE_EINVAL;
    if (ctx->T.ext_id) return fail(ctx, GPUBPE_EINVAL, "token-level merges need token ids below 2^24");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CK(cudaSetDevice(ctx->device));
    if (n_seqs == 0) return GPUBPE_OK;
    uint64_t max_len = 0;
    for (uint64_t i = 0; i < n_seqs; ++i) {
        if (h_offs[i + 1] < h_offs[i]) return fail(ctx, GPUBPE_EINVAL, "offsets decrease at %llu", (unsigned long long)i);
        max_len = std::max<uint64_t>(max_len, h_offs[i + 1] - h_offs[i]);
    }
    if (max_len && (!d_tokens || !d_out)) return fail(ctx, GPUBPE_EINVAL, "null token pointer");
    if (max_len >= (1ull << 31)) return fail(ctx, GPUBPE_EINVAL, "sequence too long for the CTA engine");
    const uint64_t per_cta = (ENGINE_BYTES(max_len) + 15) / 16 * 4;  // words
    uint64_t grid = std::min<uint64_t>(n_seqs, (uint64_t)ctx->num_sms * 2);
    while (grid > 1 && grid * per_cta * 4 > (2ull << 30)) grid >>= 1;  // arena <= 2 GiB
    int rc;
    if ((rc = ensure(ctx, ctx->ws_arena, grid * per_cta * 4, false))) return rc;
    if ((rc = ensure(ctx, ctx->mt_offs, (n_seqs + 1) * 8, false))) return rc;
    if ((rc = ensure(ctx, ctx->mt_counts, n_seqs * 8, false))) return rc;
    CK(cudaMemcpyAsync(ctx->mt_offs.p, h_offs, (n_seqs + 1) * 8, cudaMemcpyHostToDevice, s));
    MergeParams Q{};
    Q.T = ctx->T;
    Q.tok = d_tokens;
    Q.offs = static_cast<const unsigned long long *>(ctx->mt_offs.p);
    Q.n_seqs = n_seqs;
    Q.arena = static_cast<uint32_t *>(ctx->ws_arena.p);
    Q.arena_words_per_cta = per_cta;
    Q.out = d_out;
    Q.counts = static_cast<unsigned long long *>(ctx->mt_counts.p);
    Q.strict = ((ctx->flags & GPUBPE_F_STRICT) || !ctx->T.well_formed) ? 1 : 0;
    Q.n_ids = ctx->n_ids;
    Q.trace = reinterpret_cast<unsigned long long *>(d_trace);
    Q.fault_seq = fault_seq;
    CK(launch_merge_tokens(Q, (int)grid, s));
    CK(cudaMemcpyAsync(h_counts, ctx->mt_counts.p, n_seqs * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (uint64_t i = 0; i < n_seqs; ++i)
        if (h_counts[i] == ~0ull)
            return fail(ctx, GPUBPE_EINVAL, "sequence %llu holds a token id the merge table does not cover",
                        (unsigned long long)i);
    return GPUBPE_OK;
}

extern "C" __attribute__((visibility("default"))) int gpubpe_merge_tokens(gpubpe_ctx *ctx, const uint32_t *d_tokens,
                                                                           const uint64_t *h_offs, uint64_t n_seqs,
                                                                           uint32_t *d_out, uint64_t *h_counts,
                                                                           void *stream) {
    return merge_tokens(ctx, d_tokens, h_offs, n_seqs, d_out, h_counts, nullptr, -1, stream);
}

extern "C" __attribute__((visibility("default"))) int gpubpe_merge_tokens_ex(
    gpubpe_ctx *ctx, const uint32_t *d_tokens, const uint64_t *h_offs, uint64_t n_seqs, uint32_t *d_out,
    uint64_t *h_counts, uint64_t *d_trace, int64_t fault_seq, void *stream) {
    if (ctx && (fault_seq < -1 || (fault_seq >= 0 && (uint64_t)fault_seq >= n_seqs)))
        return fail(ctx, GPUBPE_EINVAL, "fault_seq %lld outside [-1, %llu)", (long long)fault_seq,
                    (unsigned long long)n_seqs);
    return merge_tokens(ctx, d_tokens, h_offs, n_seqs, d_out, h_counts, d_trace, fault_seq, stream);
}

extern "C" __attribute__((visibility("default"))) int gpubpe_eval_pairs(gpubpe_ctx *ctx, const uint32_t *d_tokens,
                                                                         uint64_t n, uint64_t *h_result,
                                                                         void *stream) {
    if (!ctx || !h_result || (n && !d_tokens)) return GPUBPE_EINVAL;
    if (ctx->T.ext_id) return fail(ctx, GPUBPE_EINVAL, "eval_pairs needs ids < 2^24");
    if (n >= (1ull << 32)) return fail(ctx, GPUBPE_EINVAL, "sequence too long for eval_pairs");
    h_result[0] = ~0ull;
    if (n < 2) return GPUBPE_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CK(cudaSetDevice(ctx->device));
    int rc;
    if ((rc = ensure(ctx, ctx->mt_counts, 3 * 8, false))) return rc;
    unsigned long long *d_res = static_cast<unsigned long long *>(ctx->mt_counts.p);
    CK(launch_eval_pairs(ctx->T, d_tokens, n, d_res, s));
    CK(cudaMemcpyAsync(h_result, d_res, 3 * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return GPUBPE_OK;
}

extern "C" __attribute__((visibility("default"))) int gpubpe_compact(const uint32_t *d_tokens, uint64_t n,
                                                                      uint64_t best_pos, uint32_t new_token,
                                                                      uint32_t *d_out, int method, void *stream) {
    if (n < 2 || best_pos >= n - 1 || !d_tokens || !d_out || (method != 0 && method != 1)) return GPUBPE_EINVAL;
    return launch_compact(d_tokens, n, best_pos, new_token, d_out, method, static_cast<cudaStream_t>(stream)) ==
                   cudaSuccess
               ? GPUBPE_OK
               : GPUBPE_ECUDA;
}

extern "C" __attribute__((visibility("default"))) int gpubpe_lookup_keys(gpubpe_ctx *ctx, const uint64_t *d_keys,
                                                                          uint64_t m, uint8_t *d_hit, uint64_t *d_vals,
                                                                          void *stream) {
    if (!ctx || (m && (!d_keys || !d_hit || !d_vals))) return GPUBPE_EINVAL;
    if (ctx->T.ext_id) return fail(ctx, GPUBPE_EINVAL, "lookup_keys needs ids < 2^24");
    CK(cudaSetDevice(ctx->device));
    CK(launch_lookup_keys(ctx->T, reinterpret_cast<const unsigned long long *>(d_keys), m, d_hit,
                          reinterpret_cast<unsigned long long *>(d_vals), static_cast<cudaStream_t>(stream)));
    return GPUBPE_OK;
}

extern "C" __attribute__((visibility("default"))) int gpubpe_junction_bits(gpubpe_ctx *ctx, uint32_t *h_out) {
    if (!ctx || !h_out) return GPUBPE_EINVAL;
    if (ctx->h_jbits.size() != 2048) return fail(ctx, GPUBPE_EINVAL, "context has no junction bitmap");
    memcpy(h_out, ctx->h_jbits.data(), 2048 * sizeof(uint32_t));
    return GPUBPE_OK;
}

extern "C" __attribute__((visibility("default"))) int gpubpe_launches_per_encode(void) { return 1; }

extern "C" __attribute__((visibility("default"))) int gpubpe_lookup_pairs(gpubpe_ctx *ctx, const uint32_t *d_left, const uint32_t *d_right,
                                   uint64_t n, uint32_t *d_new, uint32_t *d_rank, void *stream) {
    if (!ctx) return GPUBPE_EINVAL;
    if (ctx->T.ext_id) return fail(ctx, GPUBPE_EINVAL, "lookup_pairs needs ids < 2^24");
    CK(cudaSetDevice(ctx->device));
    CK(launch_lookup(ctx->T, d_left, d_right, n, d_new, d_rank, static_cast<cudaStream_t>(stream)));
    return GPUBPE_OK;
}

extern "C" __attribute__((visibility("default"))) int gpubpe_set_profiling(gpubpe_ctx *ctx, int on) {
    if (!ctx) return GPUBPE_EINVAL;
    CK(cudaSetDevice(ctx->device));
    if (on && !ctx->ev[0])
        for (auto &e : ctx->ev) CK(cudaEventCreate(&e));
    ctx->profiling = on != 0;
    return GPUBPE_OK;
}

extern "C" __attribute__((visibility("default"))) int gpubpe_kernel_ms(gpubpe_ctx *ctx, float *ms, int n) {
    if (!ctx || !ms) return GPUBPE_EINVAL;
    if (!ctx->timed) return fail(ctx, GPUBPE_EINVAL, "no profiled encode yet (gpubpe_set_profiling)");
    CK(cudaEventSynchronize(ctx->ev[1]));
    if (n >= 1) CK(cudaEventElapsedTime(&ms[0], ctx->ev[0], ctx->ev[1]));
    return GPUBPE_OK;
}

extern "C" __attribute__((visibility("default"))) const char *gpubpe_last_error(gpubpe_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

extern "C" __attribute__((visibility("default"))) void gpubpe_ctx_destroy(gpubpe_ctx *ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();
    if (ctx->tables) cudaFree(ctx->tables);
    for (DevBuf *b : {&ctx->ws_state, &ctx->ws_status, &ctx->ws_recs, &ctx->ws_scratch, &ctx->ws_tiles,
                      &ctx->ws_arena, &ctx->io_dev, &ctx->ws_gscr, &ctx->ws_glist})
        if (b->p) cudaFree(b->p);
    if (ctx->pin) cudaFreeHost(ctx->pin);
    for (auto &S : ctx->ss) {
        if (S.pin_in) cudaFreeHost(S.pin_in);
        if (S.pin_out) cudaFreeHost(S.pin_out);
        if (S.dev_in.p) cudaFree(S.dev_in.p);
        if (S.dev_out.p) cudaFree(S.dev_out.p);
        for (cudaEvent_t e : {S.ev_h2d, S.ev_done, S.ev_d2h})
            if (e) cudaEventDestroy(e);
    }
    if (ctx->s_copy) cudaStreamDestroy(ctx->s_copy);
    if (ctx->s_d2h) cudaStreamDestroy(ctx->s_d2h);
    if (ctx->h_state_ss) cudaFreeHost(ctx->h_state_ss);
    if (ctx->d_vinfo) cudaFree(ctx->d_vinfo);
    if (ctx->d_vblob) cudaFree(ctx->d_vblob);
    if (ctx->d_vrec) cudaFree(ctx->d_vrec);
    if (ctx->d_vlen) cudaFree(ctx->d_vlen);
    if (ctx->d_vlong) cudaFree(ctx->d_vlong);
    for (DevBuf *b : {&ctx->dec_state, &ctx->dec_status, &ctx->dec_tiles, &ctx->pt_bits, &ctx->mt_offs, &ctx->mt_counts})
        if (b->p) cudaFree(b->p);
    if (ctx->d_pt_classes) cudaFree(ctx->d_pt_classes);
    for (auto &e : ctx->io_ev)
        if (e) cudaEventDestroy(e);
    if (ctx->h_state) cudaFreeHost(ctx->h_state);
    if (ctx->h_mirror) cudaFreeHost(ctx->h_mirror);
    if (ctx->h_tag) cudaFreeHost(ctx->h_tag);
    if (ctx->d_arrive) cudaFree(ctx->d_arrive);
    for (auto &e : ctx->ev)
        if (e) cudaEventDestroy(e);
    delete ctx;
}
