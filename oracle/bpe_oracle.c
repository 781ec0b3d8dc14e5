/*
 * bpe_oracle.c -- CPU restatement of the reference's encode path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("port") for bench.py; it is never linked into, loaded by, or
 * called from the product path (paper_2603_02597_b200/).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may use it.
 *
 * What it restates (all paths relative to /root/reference/pkg):
 *   - merge table: 64-bit packed key (left<<32)|right, value (new<<32)|rank,
 *     murmur3 fmix64 hash, power-of-two linear probing at <= 50% load, empty
 *     key 2^64-1, DuplicatePair / ReservedKey errors
 *       src/lanebpe/merge_table.py:28-57 (constants, pack, _mix64)
 *       src/lanebpe/merge_table.py:155-168 (PackedPairTable.lookup)
 *       src/lanebpe/merge_table.py:246-278 (build_table)
 *   - the sequential engine: heap of (rank, pos, left, right, new) over a
 *     doubly linked list, stale entries skipped by id check
 *       src/lanebpe/engines.py:269-335 (sequential_bpe)
 *   - the batch pipeline: per-byte base ids, fixed-offset chunking at
 *     chunk_budget only when len > max_seq_len, chunks concatenated in order
 *       src/lanebpe/chunker.py:42-53 (chunk_tokens)
 *       src/lanebpe/chunker.py:95-98 (Tokenizer.encode)
 *       src/lanebpe/chunker.py:110-187 (tokenize_batch)
 *   The reference runs chunks on a ThreadPoolExecutor (chunker.py:157-164);
 *   here chunks are spread over pthreads, which cannot change the output.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ERR_DUPLICATE 1
#define ORC_ERR_RESERVED 2
#define ORC_ERR_NOMEM 3
#define ORC_ERR_ARG 4

static const uint64_t EMPTY = 0xFFFFFFFFFFFFFFFFull;

static inline uint64_t fmix64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xFF51AFD7ED558CCDull;
    x ^= x >> 33;
    x *= 0xC4CEB9FE1A85EC53ull;
    x ^= x >> 33;
    return x;
}

typedef struct orc_table {
    uint64_t *keys;
    uint64_t *vals;
    uint64_t mask;
    uint64_t capacity;
    uint64_t count;
} orc_table;

void orc_table_free(orc_table *t) {
    if (!t) return;
    free(t->keys);
    free(t->vals);
    free(t);
}

/* Build from rule arrays; err_index receives the offending rule on error. */
int orc_table_build(const uint32_t *left, const uint32_t *right, const uint32_t *rank,
                    const uint32_t *new_tok, uint64_t n, orc_table **out,
                    uint64_t *err_index) {
    uint64_t cap = 1;
    while (cap < 2 * n) cap <<= 1;
    orc_table *t = (orc_table *)calloc(1, sizeof(orc_table));
    if (!t) return ORC_ERR_NOMEM;
    t->keys = (uint64_t *)malloc(cap * sizeof(uint64_t));
    t->vals = (uint64_t *)calloc(cap, sizeof(uint64_t));
    if (!t->keys || !t->vals) {
        orc_table_free(t);
        return ORC_ERR_NOMEM;
    }
    memset(t->keys, 0xFF, cap * sizeof(uint64_t));
    t->capacity = cap;
    t->mask = cap - 1;
    t->count = n;
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t key = ((uint64_t)left[i] << 32) | right[i];
        if (key == EMPTY) {
            if (err_index) *err_index = i;
            orc_table_free(t);
            return ORC_ERR_RESERVED;
        }
        uint64_t idx = fmix64(key) & t->mask;
        for (;;) {
            if (t->keys[idx] == EMPTY) break;
            if (t->keys[idx] == key) {
                if (err_index) *err_index = i;
                orc_table_free(t);
                return ORC_ERR_DUPLICATE;
            }
            idx = (idx + 1) & t->mask;
        }
        t->keys[idx] = key;
        t->vals[idx] = ((uint64_t)new_tok[i] << 32) | rank[i];
    }
    *out = t;
    return ORC_OK;
}

/* 1 on hit (value written), 0 on miss. */
static inline int table_lookup(const orc_table *t, uint32_t l, uint32_t r, uint64_t *val) {
    uint64_t key = ((uint64_t)l << 32) | r;
    if (key == EMPTY || t->capacity == 0) return 0;
    uint64_t idx = fmix64(key) & t->mask;
    for (;;) {
        uint64_t k = t->keys[idx];
        if (k == key) {
            *val = t->vals[idx];
            return 1;
        }
        if (k == EMPTY) return 0;
        idx = (idx + 1) & t->mask;
    }
}

int orc_table_lookup(const orc_table *t, uint32_t l, uint32_t r, uint32_t *new_tok,
                     uint32_t *rank) {
    uint64_t v;
    if (!table_lookup(t, l, r, &v)) return 0;
    *new_tok = (uint32_t)(v >> 32);
    *rank = (uint32_t)v;
    return 1;
}

/* ---------------------------------------------------------------- heap */

typedef struct {
    uint32_t rank;
    uint64_t pos;
    uint32_t l, r, nw;
} hent;

static inline int hless(const hent *a, const hent *b) {
    if (a->rank != b->rank) return a->rank < b->rank;
    if (a->pos != b->pos) return a->pos < b->pos;
    if (a->l != b->l) return a->l < b->l;
    if (a->r != b->r) return a->r < b->r;
    return a->nw < b->nw;
}

typedef struct {
    hent *v;
    uint64_t n, cap;
} heap_t;

static int heap_push(heap_t *h, hent e) {
    if (h->n == h->cap) {
        uint64_t nc = h->cap ? h->cap * 2 : 64;
        hent *nv = (hent *)realloc(h->v, nc * sizeof(hent));
        if (!nv) return -1;
        h->v = nv;
        h->cap = nc;
    }
    uint64_t i = h->n++;
    while (i > 0) {
        uint64_t p = (i - 1) / 2;
        if (!hless(&e, &h->v[p])) break;
        h->v[i] = h->v[p];
        i = p;
    }
    h->v[i] = e;
    return 0;
}

static hent heap_pop(heap_t *h) {
    hent top = h->v[0];
    hent last = h->v[--h->n];
    uint64_t i = 0, n = h->n;
    for (;;) {
        uint64_t c = 2 * i + 1;
        if (c >= n) break;
        if (c + 1 < n && hless(&h->v[c + 1], &h->v[c])) c++;
        if (!hless(&h->v[c], &last)) break;
        h->v[i] = h->v[c];
        i = c;
    }
    if (n) h->v[i] = last;
    return top;
}

/*
 * sequential_bpe restated (engines.py:269-335).  tokens[0..n) -> out, returns
 * output length; *passes += merges applied; if trace != NULL the rank of every
 * merge is appended (trace must hold n entries).  Returns UINT64_MAX on OOM.
 */
uint64_t orc_sequential_bpe(const orc_table *t, const uint32_t *tokens, uint64_t n,
                            uint32_t *out, uint64_t *passes, uint32_t *trace) {
    if (n < 2) {
        for (uint64_t i = 0; i < n; ++i) out[i] = tokens[i];
        return n;
    }
    uint32_t *ids = (uint32_t *)malloc(n * sizeof(uint32_t));
    int64_t *nxt = (int64_t *)malloc(n * sizeof(int64_t));
    int64_t *prv = (int64_t *)malloc(n * sizeof(int64_t));
    uint8_t *alive = (uint8_t *)malloc(n);
    heap_t h = {0, 0, 0};
    uint64_t merges = 0;
    if (!ids || !nxt || !prv || !alive) goto oom;
    for (uint64_t i = 0; i < n; ++i) {
        ids[i] = tokens[i];
        nxt[i] = (i + 1 < n) ? (int64_t)(i + 1) : -1;
        prv[i] = (int64_t)i - 1;
        alive[i] = 1;
    }
    for (uint64_t i = 0; i + 1 < n; ++i) {
        uint64_t v;
        if (table_lookup(t, ids[i], ids[i + 1], &v)) {
            hent e = {(uint32_t)v, i, ids[i], ids[i + 1], (uint32_t)(v >> 32)};
            if (heap_push(&h, e)) goto oom;
        }
    }
    while (h.n) {
        hent e = heap_pop(&h);
        uint64_t pos = e.pos;
        if (!alive[pos]) continue;
        int64_t right = nxt[pos];
        if (right == -1 || ids[pos] != e.l || ids[right] != e.r) continue;
        ids[pos] = e.nw;
        alive[right] = 0;
        int64_t after = nxt[right];
        nxt[pos] = after;
        if (after != -1) prv[after] = (int64_t)pos;
        if (trace) trace[merges] = e.rank;
        merges++;
        int64_t before = prv[pos];
        uint64_t v;
        if (before != -1 && table_lookup(t, ids[before], e.nw, &v)) {
            hent ne = {(uint32_t)v, (uint64_t)before, ids[before], e.nw, (uint32_t)(v >> 32)};
            if (heap_push(&h, ne)) goto oom;
        }
        if (after != -1 && table_lookup(t, e.nw, ids[after], &v)) {
            hent ne = {(uint32_t)v, pos, e.nw, ids[after], (uint32_t)(v >> 32)};
            if (heap_push(&h, ne)) goto oom;
        }
    }
    {
        uint64_t k = 0;
        for (uint64_t i = 0; i < n; ++i)
            if (alive[i]) out[k++] = ids[i];
        free(ids); free(nxt); free(prv); free(alive); free(h.v);
        if (passes) *passes += merges;
        return k;
    }
oom:
    free(ids); free(nxt); free(prv); free(alive); free(h.v);
    return UINT64_MAX;
}

/* ------------------------------------------------------------- batch path */

typedef struct {
    uint64_t in_off; /* byte offset of the chunk in the packed input */
    uint64_t len;
    uint64_t out_len;
} chunk_t;

typedef struct {
    const orc_table *t;
    const uint32_t *base;
    const uint8_t *bytes;
    chunk_t *chunks;
    uint64_t n_chunks;
    uint32_t *scratch; /* per-byte slots: chunk k writes [in_off, in_off+out_len) */
    volatile uint64_t next;
    uint64_t passes;
    int failed;
    pthread_mutex_t mu;
} batch_job;

static void *batch_worker(void *arg) {
    batch_job *j = (batch_job *)arg;
    uint32_t *tmp = NULL;
    uint64_t tmp_cap = 0, my_passes = 0;
    for (;;) {
        uint64_t k = __atomic_fetch_add(&j->next, 1, __ATOMIC_RELAXED);
        if (k >= j->n_chunks) break;
        chunk_t *c = &j->chunks[k];
        if (c->len > tmp_cap) {
            free(tmp);
            tmp_cap = c->len;
            tmp = (uint32_t *)malloc(tmp_cap * sizeof(uint32_t));
            if (!tmp) { j->failed = 1; break; }
        }
        for (uint64_t i = 0; i < c->len; ++i) tmp[i] = j->base[j->bytes[c->in_off + i]];
        uint64_t m = orc_sequential_bpe(j->t, tmp, c->len, j->scratch + c->in_off, &my_passes, NULL);
        if (m == UINT64_MAX) { j->failed = 1; break; }
        c->out_len = m;
    }
    free(tmp);
    pthread_mutex_lock(&j->mu);
    j->passes += my_passes;
    pthread_mutex_unlock(&j->mu);
    return NULL;
}

/*
 * tokenize_batch restated: bytes[doc_offs[d] .. doc_offs[d+1]) for d < n_docs.
 * out_ids must hold doc_offs[n_docs] entries; out_offs n_docs+1.  Returns
 * ORC_OK and the total merge count in *passes.
 */
int orc_tokenize_batch(const orc_table *t, const uint32_t base_ids[256], const uint8_t *bytes,
                       const int64_t *doc_offs, uint64_t n_docs, uint64_t max_seq_len,
                       uint64_t chunk_budget, int threads, uint32_t *out_ids,
                       int64_t *out_offs, uint64_t *passes) {
    if (chunk_budget < 2 || (n_docs && doc_offs[0] != 0)) return ORC_ERR_ARG;
    uint64_t n_chunks = 0;
    for (uint64_t d = 0; d < n_docs; ++d) {
        uint64_t len = (uint64_t)(doc_offs[d + 1] - doc_offs[d]);
        if (len == 0) continue;
        n_chunks += (len > max_seq_len) ? (len + chunk_budget - 1) / chunk_budget : 1;
    }
    uint64_t total = n_docs ? (uint64_t)(doc_offs[n_docs] - doc_offs[0]) : 0;
    chunk_t *chunks = (chunk_t *)malloc((n_chunks ? n_chunks : 1) * sizeof(chunk_t));
    uint32_t *scratch = (uint32_t *)malloc((total ? total : 1) * sizeof(uint32_t));
    if (!chunks || !scratch) {
        free(chunks); free(scratch);
        return ORC_ERR_NOMEM;
    }
    uint64_t k = 0;
    for (uint64_t d = 0; d < n_docs; ++d) {
        uint64_t s = (uint64_t)doc_offs[d], len = (uint64_t)(doc_offs[d + 1] - doc_offs[d]);
        if (len == 0) continue;
        uint64_t step = (len > max_seq_len) ? chunk_budget : len;
        for (uint64_t off = 0; off < len; off += step) {
            chunks[k].in_off = s + off;
            chunks[k].len = (len - off < step) ? len - off : step;
            chunks[k].out_len = 0;
            k++;
        }
    }
    batch_job j;
    j.t = t; j.base = base_ids; j.bytes = bytes; j.chunks = chunks; j.n_chunks = n_chunks;
    j.scratch = scratch; j.next = 0; j.passes = 0; j.failed = 0;
    pthread_mutex_init(&j.mu, NULL);
    if (threads < 1) threads = 1;
    if ((uint64_t)threads > n_chunks) threads = n_chunks ? (int)n_chunks : 1;
    if (threads == 1) {
        batch_worker(&j);
    } else {
        pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)threads);
        for (int i = 0; i < threads; ++i) pthread_create(&th[i], NULL, batch_worker, &j);
        for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
        free(th);
    }
    pthread_mutex_destroy(&j.mu);
    if (j.failed) {
        free(chunks); free(scratch);
        return ORC_ERR_NOMEM;
    }
    /* ordered assembly (chunker.py:166-179) */
    uint64_t o = 0;
    k = 0;
    for (uint64_t d = 0; d < n_docs; ++d) {
        out_offs[d] = (int64_t)o;
        uint64_t end = (uint64_t)doc_offs[d + 1];
        while (k < n_chunks && chunks[k].in_off < end) {
            memcpy(out_ids + o, scratch + chunks[k].in_off, chunks[k].out_len * sizeof(uint32_t));
            o += chunks[k].out_len;
            k++;
        }
    }
    out_offs[n_docs] = (int64_t)o;
    if (passes) *passes = j.passes;
    free(chunks); free(scratch);
    return ORC_OK;
}
