/*
 * TEST INFRASTRUCTURE ONLY -- see acz_oracle.h. Plain-C restatement of the reference
 * codec; every function cites the reference file:line it follows. Compile with
 * -ffp-contract=off (no FMA) and no -march: the reference's canonical build.
 */
#include "acz_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

enum { OK = 0, E_PARAM = 1, E_DOMAIN = 2, E_FORMAT = 3, E_DECODE = 4, E_SHAPE = 5, E_NOMEM = 7 };

static int fail(char* err, int cap, int code, const char* msg) {
    if (err && cap > 0) {
        strncpy(err, msg, (size_t)cap - 1);
        err[cap - 1] = 0;
    }
    return code;
}

void oracle_free(void* p) { free(p); }

/* ref src/codec.cpp:54-59 (CodecParams::validate) */
static int validate_params(double eb, uint32_t radius, char* err, int cap) {
    if (!(eb > 0.0) || !isfinite(eb)) return fail(err, cap, E_PARAM, "error bound must be positive");
    if (radius < 2 || radius > (1u << 24) || (radius & (radius - 1)) != 0)
        return fail(err, cap, E_PARAM, "quant_radius must be a power of two in [2, 2^24]");
    return OK;
}

/* ref src/codec.cpp:21-34 (PlaneView) */
static void plane_view(const uint64_t* shape, int rank, uint64_t* planes, uint64_t* rows,
                       uint64_t* cols) {
    *planes = 1;
    *rows = 1;
    *cols = 1;
    if (rank == 0) return;
    if (rank == 1) {
        *cols = shape[0];
        return;
    }
    *rows = shape[rank - 2];
    *cols = shape[rank - 1];
    for (int i = 0; i + 2 < rank; ++i) *planes *= shape[i];
}

/* ref src/codec.cpp:36-50 (predict) */
static double predict(int pred, const float* plane, uint64_t cols, uint64_t r, uint64_t c) {
    const uint64_t at = r * cols + c;
    if (pred == 0) return at == 0 ? 0.0 : (double)plane[at - 1];
    double left = c > 0 ? plane[at - 1] : 0.0;
    double top = r > 0 ? plane[at - cols] : 0.0;
    double topleft = (r > 0 && c > 0) ? plane[at - cols - 1] : 0.0;
    return left + top - topleft;
}

/* ---------------------------------------------------------------- Huffman ---- */

typedef struct {
    uint64_t freq;
    uint32_t tiebreak;
} item;

static int item_less(item a, item b) {
    return a.freq != b.freq ? a.freq < b.freq : a.tiebreak < b.tiebreak;
}

static void heap_push(item* h, uint64_t* n, item v) {
    uint64_t i = (*n)++;
    h[i] = v;
    while (i > 0) {
        uint64_t p = (i - 1) / 2;
        if (!item_less(h[i], h[p])) break;
        item t = h[i];
        h[i] = h[p];
        h[p] = t;
        i = p;
    }
}

static item heap_pop(item* h, uint64_t* n) {
    item top = h[0];
    h[0] = h[--(*n)];
    uint64_t i = 0;
    for (;;) {
        uint64_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < *n && item_less(h[l], h[m])) m = l;
        if (r < *n && item_less(h[r], h[m])) m = r;
        if (m == i) break;
        item t = h[i];
        h[i] = h[m];
        h[m] = t;
        i = m;
    }
    return top;
}

static int cmp_u32(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : x > y;
}

typedef struct {
    uint32_t sym;
    uint8_t len;
} entry;

static int cmp_entry(const void* a, const void* b) {
    const entry* x = (const entry*)a;
    const entry* y = (const entry*)b;
    if (x->len != y->len) return x->len < y->len ? -1 : 1;
    return x->sym < y->sym ? -1 : x->sym > y->sym;
}

/* ---- thread helpers (the multi-threaded oracle splits work into contiguous ranges and
 * joins the results in index order, so its outputs are those of the serial loops) ---- */
typedef void (*range_fn)(void* arg, int t, int nt);
typedef struct {
    range_fn fn;
    void* arg;
    int t, nt;
} range_job;
static void* range_main(void* p) {
    range_job* j = (range_job*)p;
    j->fn(j->arg, j->t, j->nt);
    return NULL;
}
/* runs fn(arg, t, nt) for t in [0, nt) on nt threads (thread 0 is the caller) */
static void run_threads(range_fn fn, void* arg, int nt) {
    if (nt <= 1) {
        fn(arg, 0, 1);
        return;
    }
    pthread_t th[256];
    range_job jobs[256];
    if (nt > 256) nt = 256;
    int started[256] = {0};
    for (int t = 1; t < nt; ++t) {
        jobs[t] = (range_job){fn, arg, t, nt};
        started[t] = pthread_create(&th[t], NULL, range_main, &jobs[t]) == 0;
        if (!started[t]) fn(arg, t, nt);
    }
    fn(arg, 0, nt);
    for (int t = 1; t < nt; ++t)
        if (started[t]) pthread_join(th[t], NULL);
}
static void split(uint64_t n, int t, int nt, uint64_t* a, uint64_t* b) {
    *a = n * (uint64_t)t / (uint64_t)nt;
    *b = n * (uint64_t)(t + 1) / (uint64_t)nt;
}

typedef struct {
    const uint32_t* syms;
    uint64_t n;
    uint32_t mx;
    uint64_t* part; /* nt x (mx + 1) counts */
} count_job;
static void count_range(void* p, int t, int nt) {
    count_job* j = (count_job*)p;
    uint64_t a, b;
    split(j->n, t, nt, &a, &b);
    uint64_t* d = j->part + (uint64_t)t * ((uint64_t)j->mx + 1);
    for (uint64_t i = a; i < b; ++i) d[j->syms[i]]++;
}

typedef struct {
    const uint32_t* syms;
    uint64_t n;
    uint32_t* mx; /* per thread */
} max_job;
static void max_range(void* p, int t, int nt) {
    max_job* j = (max_job*)p;
    uint64_t a, b;
    split(j->n, t, nt, &a, &b);
    uint32_t m = 0;
    for (uint64_t i = a; i < b; ++i)
        if (j->syms[i] > m) m = j->syms[i];
    j->mx[t] = m;
}

/* Frequencies in ascending symbol order: ref src/huffman.cpp:110-111 (std::map). */
static int frequencies(const uint32_t* syms, uint64_t n, uint32_t** fsym, uint64_t** ffreq,
                       uint64_t* k, int nt) {
    uint32_t mx = 0;
    {
        uint32_t m[256] = {0};
        max_job mj = {syms, n, m};
        run_threads(max_range, &mj, nt);
        for (int t = 0; t < (nt > 256 ? 256 : nt); ++t)
            if (m[t] > mx) mx = m[t];
    }
    uint64_t cnt = 0;
    if (mx < (1u << 26)) {
        uint64_t* dense = calloc((size_t)mx + 1, sizeof(uint64_t));
        if (!dense) return E_NOMEM;
        uint64_t* part = NULL;
        if (nt > 1 && mx < (1u << 22))
            part = calloc((size_t)nt * ((size_t)mx + 1), sizeof(uint64_t));
        if (part) {
            count_job cj = {syms, n, mx, part};
            run_threads(count_range, &cj, nt);
            for (int t = 0; t < nt; ++t)
                for (uint64_t s2 = 0; s2 <= mx; ++s2)
                    dense[s2] += part[(uint64_t)t * ((uint64_t)mx + 1) + s2];
            free(part);
        } else {
            for (uint64_t i = 0; i < n; ++i) dense[syms[i]]++;
        }
        for (uint64_t s = 0; s <= mx; ++s) cnt += dense[s] != 0;
        *fsym = malloc(sizeof(uint32_t) * (cnt + 1));
        *ffreq = malloc(sizeof(uint64_t) * (cnt + 1));
        uint64_t j = 0;
        for (uint64_t s = 0; s <= mx; ++s)
            if (dense[s]) {
                (*fsym)[j] = (uint32_t)s;
                (*ffreq)[j++] = dense[s];
            }
        free(dense);
    } else {
        uint32_t* tmp = malloc(sizeof(uint32_t) * n);
        if (!tmp) return E_NOMEM;
        memcpy(tmp, syms, sizeof(uint32_t) * n);
        qsort(tmp, n, sizeof(uint32_t), cmp_u32);
        for (uint64_t i = 0; i < n; ++i) cnt += (i == 0 || tmp[i] != tmp[i - 1]);
        *fsym = malloc(sizeof(uint32_t) * (cnt + 1));
        *ffreq = malloc(sizeof(uint64_t) * (cnt + 1));
        uint64_t j = 0;
        for (uint64_t i = 0; i < n; ++i) {
            if (i == 0 || tmp[i] != tmp[i - 1]) {
                (*fsym)[j] = tmp[i];
                (*ffreq)[j++] = 0;
            }
            (*ffreq)[j - 1]++;
        }
        free(tmp);
    }
    *k = cnt;
    return OK;
}

/* ref src/huffman.cpp:22-72 (code_lengths): min-heap on (freq, creation index); leaves
 * created in ascending symbol order; one symbol -> length 1; depth > 64 -> DecodeError.
 * Lengths are returned per leaf (same order as fsym). */
static int code_lengths(const uint64_t* ffreq, uint64_t k, uint8_t* len, char* err, int cap) {
    if (k == 0) return OK;
    if (k == 1) {
        len[0] = 1;
        return OK;
    }
    uint64_t total = 2 * k - 1;
    int64_t* parent = malloc(sizeof(int64_t) * total);
    item* heap = malloc(sizeof(item) * k);
    if (!parent || !heap) {
        free(parent);
        free(heap);
        return E_NOMEM;
    }
    uint64_t hn = 0;
    for (uint64_t i = 0; i < k; ++i) {
        item it = {ffreq[i], (uint32_t)i};
        heap_push(heap, &hn, it);
    }
    uint64_t next = k;
    while (hn > 1) {
        item a = heap_pop(heap, &hn);
        item b = heap_pop(heap, &hn);
        parent[a.tiebreak] = (int64_t)next;
        parent[b.tiebreak] = (int64_t)next;
        item p = {a.freq + b.freq, (uint32_t)next};
        heap_push(heap, &hn, p);
        ++next;
    }
    /* Every parent has a larger index than its children: depths top-down. */
    uint32_t* depth = malloc(sizeof(uint32_t) * total);
    depth[total - 1] = 0;
    for (int64_t i = (int64_t)total - 2; i >= 0; --i) depth[i] = depth[parent[i]] + 1;
    int rc = OK;
    for (uint64_t i = 0; i < k; ++i) {
        if (depth[i] > 64) {
            rc = fail(err, cap, E_DECODE, "huffman code length exceeds 64 bits");
            break;
        }
        len[i] = (uint8_t)depth[i];
    }
    free(depth);
    free(parent);
    free(heap);
    return rc;
}

/* ref src/huffman.cpp:75-86 (canonical_codes) */
static void canonical_codes(const entry* book, uint64_t k, uint64_t* codes) {
    uint64_t code = 0;
    uint8_t prev = 0;
    for (uint64_t i = 0; i < k; ++i) {
        code <<= (book[i].len - prev);
        codes[i] = code;
        ++code;
        prev = book[i].len;
    }
}

/* ref src/huffman.cpp:107-135 (huffman_encode); BitWriter :88-103 (MSB-first). */
typedef struct {
    const uint32_t* syms;
    uint64_t n;
    const uint64_t* code_of_sym; /* dense: symbol -> code */
    const uint8_t* len_of_sym;   /* dense: symbol -> length */
    uint64_t* start;             /* per thread: first bit (filled by the caller) */
    uint64_t* nbits;             /* per thread: bit count (first pass) */
    uint8_t** local;             /* per thread: private bytes from byte start[t] / 8 */
    int pass;
    int nomem;
} pack_job;
/* MSB-first packing of a contiguous symbol range into a private buffer aligned like the
 * shared stream (its first byte is byte start/8 of the stream): ref BitWriter,
 * src/huffman.cpp:88-103, loop :127-131. */
static void pack_range(void* p, int t, int nt) {
    pack_job* j = (pack_job*)p;
    uint64_t a, b;
    split(j->n, t, nt, &a, &b);
    if (j->pass == 0) {
        uint64_t c = 0;
        for (uint64_t i = a; i < b; ++i) c += j->len_of_sym[j->syms[i]];
        j->nbits[t] = c;
        return;
    }
    const uint64_t s0 = j->start[t];
    const uint64_t nbytes = ((s0 & 7) + j->nbits[t] + 7) / 8 + 1;
    uint8_t* out = calloc((size_t)nbytes, 1);
    j->local[t] = out;
    if (!out) {
        j->nomem = 1;
        return;
    }
    uint64_t pos = s0 & 7;
    for (uint64_t i = a; i < b; ++i) {
        const uint32_t s2 = j->syms[i];
        const uint64_t code = j->code_of_sym[s2];
        for (int bit = j->len_of_sym[s2] - 1; bit >= 0; --bit, ++pos)
            if ((code >> bit) & 1) out[pos >> 3] |= (uint8_t)(0x80u >> (pos & 7));
    }
}

static int huffman_encode_impl(const uint32_t* syms, uint64_t n, uint32_t* book_size,
                               uint32_t** book_sym, uint8_t** book_len, uint8_t** bits,
                               uint64_t* bit_length, char* err, int cap, int nt) {
    *book_size = 0;
    *book_sym = NULL;
    *book_len = NULL;
    *bits = NULL;
    *bit_length = 0;
    if (n == 0) return OK;
    uint32_t* fsym = NULL;
    uint64_t* ffreq = NULL;
    uint64_t k = 0;
    int rc = frequencies(syms, n, &fsym, &ffreq, &k, nt);
    if (rc) return fail(err, cap, rc, "out of memory");
    uint8_t* len = malloc(k);
    rc = code_lengths(ffreq, k, len, err, cap);
    if (rc) {
        free(fsym);
        free(ffreq);
        free(len);
        return rc;
    }
    entry* book = malloc(sizeof(entry) * k);
    for (uint64_t i = 0; i < k; ++i) {
        book[i].sym = fsym[i];
        book[i].len = len[i];
    }
    qsort(book, k, sizeof(entry), cmp_entry);
    uint64_t* codes = malloc(sizeof(uint64_t) * k);
    canonical_codes(book, k, codes);
    /* symbol -> (code, len) lookup via binary search over fsym (ascending) */
    uint64_t* code_of = malloc(sizeof(uint64_t) * k);
    uint8_t* len_of = malloc(k);
    for (uint64_t i = 0; i < k; ++i) {
        uint64_t lo = 0, hi = k;
        while (lo < hi) {
            uint64_t mid = (lo + hi) / 2;
            if (fsym[mid] < book[i].sym) lo = mid + 1; else hi = mid;
        }
        code_of[lo] = codes[i];
        len_of[lo] = book[i].len;
    }
    uint64_t total_bits = 0;
    for (uint64_t i = 0; i < k; ++i) total_bits += ffreq[i] * len_of[i];
    uint8_t* out = calloc((size_t)((total_bits + 7) / 8) + 1, 1);
    uint64_t pos = 0;
    uint64_t prev_sym_idx = 0;
    const uint32_t mxs = fsym[k - 1];
    uint64_t* dcode = NULL;
    uint8_t* dlen = NULL;
    if (nt > 1 && mxs < (1u << 26)) {
        dcode = calloc((size_t)mxs + 1, sizeof(uint64_t));
        dlen = calloc((size_t)mxs + 1, 1);
    }
    if (dcode && dlen) {
        /* threaded packing: per-range bit counts, exclusive prefix, private aligned
         * buffers OR-ed into the stream in range order (bytes shared by two ranges
         * receive both ranges' bits) */
        for (uint64_t i = 0; i < k; ++i) {
            dcode[fsym[i]] = code_of[i];
            dlen[fsym[i]] = len_of[i];
        }
        uint64_t start[256], nbits[256];
        uint8_t* local[256] = {0};
        int ntt = nt > 256 ? 256 : nt;
        pack_job pj = {syms, n, dcode, dlen, start, nbits, local, 0, 0};
        run_threads(pack_range, &pj, ntt);
        uint64_t acc = 0;
        for (int t = 0; t < ntt; ++t) {
            start[t] = acc;
            acc += nbits[t];
        }
        pj.pass = 1;
        run_threads(pack_range, &pj, ntt);
        for (int t = 0; t < ntt; ++t) {
            if (local[t]) {
                const uint64_t b0 = start[t] >> 3;
                const uint64_t nb = ((start[t] & 7) + nbits[t] + 7) / 8;
                for (uint64_t i = 0; i < nb; ++i) out[b0 + i] |= local[t][i];
            }
            free(local[t]);
        }
        pos = acc;
        free(dcode);
        free(dlen);
        if (pj.nomem) {
            free(out);
            free(fsym);
            free(ffreq);
            free(len);
            free(book);
            free(codes);
            free(code_of);
            free(len_of);
            return fail(err, cap, E_NOMEM, "out of memory");
        }
    } else {
    free(dcode);
    free(dlen);
    for (uint64_t i = 0; i < n; ++i) {
        uint32_t s = syms[i];
        uint64_t j;
        if (fsym[prev_sym_idx] == s) {
            j = prev_sym_idx;
        } else {
            uint64_t lo = 0, hi = k;
            while (lo < hi) {
                uint64_t mid = (lo + hi) / 2;
                if (fsym[mid] < s) lo = mid + 1; else hi = mid;
            }
            j = lo;
            prev_sym_idx = j;
        }
        uint64_t code = code_of[j];
        int l = len_of[j];
        for (int b = l - 1; b >= 0; --b, ++pos)
            if ((code >> b) & 1) out[pos >> 3] |= (uint8_t)(0x80u >> (pos & 7));
    }
    }
    *book_size = (uint32_t)k;
    *book_sym = malloc(sizeof(uint32_t) * k);
    *book_len = malloc(k);
    for (uint64_t i = 0; i < k; ++i) {
        (*book_sym)[i] = book[i].sym;
        (*book_len)[i] = book[i].len;
    }
    *bits = out;
    *bit_length = pos;
    free(fsym);
    free(ffreq);
    free(len);
    free(book);
    free(codes);
    free(code_of);
    free(len_of);
    return OK;
}

int oracle_huffman_encode(const uint32_t* syms, uint64_t n, uint32_t* book_size,
                          uint32_t** book_sym, uint8_t** book_len, uint8_t** bits,
                          uint64_t* bit_length, char* err, int errcap) {
    return huffman_encode_impl(syms, n, book_size, book_sym, book_len, bits, bit_length, err,
                               errcap, 1);
}

/* ref src/huffman.cpp:137-189 (huffman_decode), bit-serial canonical decode. */
int oracle_huffman_decode(const uint32_t* book_sym, const uint8_t* book_len,
                          uint32_t book_size, const uint8_t* bits, uint64_t bit_length,
                          uint64_t count, uint32_t* out, char* err, int cap) {
    if (count == 0) return OK;
    if (book_size == 0) return fail(err, cap, E_DECODE, "empty codebook");
    for (uint32_t i = 1; i < book_size; ++i) {
        uint8_t la = book_len[i - 1], lb = book_len[i];
        if (la > lb || (la == lb && book_sym[i - 1] >= book_sym[i]))
            return fail(err, cap, E_DECODE, "codebook entries are not in canonical order");
    }
    for (uint32_t i = 0; i < book_size; ++i)
        if (book_len[i] == 0 || book_len[i] > 64)
            return fail(err, cap, E_DECODE, "invalid code length in codebook");
    uint64_t first_code[65] = {0}, first_index[65] = {0}, cnt[65] = {0};
    {
        uint64_t code = 0;
        uint8_t prev = 0;
        for (uint32_t i = 0; i < book_size; ++i) {
            code <<= (book_len[i] - prev);
            uint8_t l = book_len[i];
            if (cnt[l] == 0) {
                first_code[l] = code;
                first_index[l] = i;
            }
            cnt[l]++;
            ++code;
            prev = l;
        }
    }
    uint64_t pos = 0;
    for (uint64_t o = 0; o < count; ++o) {
        uint64_t acc = 0;
        unsigned len = 0;
        for (;;) {
            if (pos >= bit_length) return fail(err, cap, E_DECODE, "truncated bitstream");
            uint64_t bit = (bits[pos >> 3] >> (7 - (pos & 7))) & 1;
            ++pos;
            acc = (acc << 1) | bit;
            ++len;
            if (len > 64) return fail(err, cap, E_DECODE, "no codeword matches bitstream");
            if (cnt[len] != 0 && acc >= first_code[len] && acc < first_code[len] + cnt[len]) {
                out[o] = book_sym[first_index[len] + (acc - first_code[len])];
                break;
            }
        }
    }
    return OK;
}

/* ------------------------------------------------------------------ bytes ---- */
/* ref include/acz/bytes.hpp:15-123 (little-endian packing) */
typedef struct {
    uint8_t* p;
    uint64_t n, cap;
} wbuf;

static void w_raw(wbuf* w, const void* src, uint64_t k) {
    if (w->n + k > w->cap) {
        uint64_t nc = (w->cap * 2 > w->n + k) ? w->cap * 2 : w->n + k + 64;
        w->p = realloc(w->p, (size_t)nc);
        w->cap = nc;
    }
    if (k) memcpy(w->p + w->n, src, (size_t)k);
    w->n += k;
}
static void w_uint(wbuf* w, uint64_t v, int bytes) {
    uint8_t b[8];
    for (int i = 0; i < bytes; ++i) b[i] = (uint8_t)(v >> (8 * i));
    w_raw(w, b, (uint64_t)bytes);
}

typedef struct {
    const uint8_t* p;
    uint64_t n, pos;
    int bad;
} rbuf;

static uint64_t r_uint(rbuf* r, int bytes) {
    if (r->bad || r->pos + (uint64_t)bytes > r->n) {
        r->bad = 1;
        return 0;
    }
    uint64_t v = 0;
    for (int i = 0; i < bytes; ++i) v |= (uint64_t)r->p[r->pos + i] << (8 * i);
    r->pos += (uint64_t)bytes;
    return v;
}

/* ------------------------------------------------------------------ codec ---- */

/* The quantise loop of ref src/codec.cpp:76-104 over planes [pl0, pl1): symbols, chain
 * values and this range's outliers (flat order). Planes are independent (the predictor
 * resets at every plane start, src/codec.cpp:17-20), so ranges run on separate threads and
 * their outlier lists concatenate in range order. */
typedef struct {
    const float* x;
    uint64_t planes, rows, cols;
    double eb;
    int64_t R;
    int predictor;
    uint32_t* symbols;
    float* recon_all;
    struct qpart {
        uint64_t n_out, ocap;
        uint64_t* oidx;
        float* oval;
        int nomem;
    } part[256];
} quant_job;

static void quantise_range(void* p, int t, int nt) {
    quant_job* j = (quant_job*)p;
    struct qpart* o = &j->part[t];
    uint64_t pl0, pl1;
    split(j->planes, t, nt, &pl0, &pl1);
    const uint64_t rows = j->rows, cols = j->cols;
    const double eb = j->eb, step = 2.0 * eb;
    const int64_t R = j->R;
    float* recon = malloc(sizeof(float) * rows * cols);
    o->ocap = 16;
    o->oidx = malloc(sizeof(uint64_t) * o->ocap);
    o->oval = malloc(sizeof(float) * o->ocap);
    if (!recon || !o->oidx || !o->oval) {
        o->nomem = 1;
        free(recon);
        return;
    }
    uint64_t flat = pl0 * rows * cols;
    for (uint64_t pl = pl0; pl < pl1; ++pl) {
        for (uint64_t r = 0; r < rows; ++r) {
            for (uint64_t c = 0; c < cols; ++c, ++flat) {
                const double orig = j->x[flat];
                const double pred = predict(j->predictor, recon, cols, r, c);
                const double q = round((orig - pred) / step); /* ties away from zero */
                float value;
                uint32_t sym = 0;
                if (fabs(q) < (double)R) {
                    const float cand = (float)(pred + q * step);
                    if (isfinite(cand) && fabs(orig - (double)cand) <= eb) {
                        sym = (uint32_t)((int64_t)q + R);
                        value = cand;
                    } else {
                        value = j->x[flat];
                    }
                } else {
                    value = j->x[flat];
                }
                if (sym == 0) {
                    if (o->n_out == o->ocap) {
                        o->ocap *= 2;
                        uint64_t* ni = realloc(o->oidx, sizeof(uint64_t) * o->ocap);
                        float* nv = realloc(o->oval, sizeof(float) * o->ocap);
                        if (ni) o->oidx = ni;
                        if (nv) o->oval = nv;
                        if (!ni || !nv) {
                            o->nomem = 1;
                            free(recon);
                            return;
                        }
                    }
                    o->oidx[o->n_out] = flat;
                    o->oval[o->n_out++] = j->x[flat];
                }
                j->symbols[flat] = sym;
                j->recon_all[flat] = value;
                recon[r * cols + c] = value;
            }
        }
    }
    free(recon);
}

typedef struct {
    const float* x;
    uint64_t n;
    int bad[256];
} finite_job;
static void finite_range(void* p, int t, int nt) {
    finite_job* j = (finite_job*)p;
    uint64_t a, b;
    split(j->n, t, nt, &a, &b);
    for (uint64_t i = a; i < b; ++i)
        if (!isfinite(j->x[i])) {
            j->bad[t] = 1;
            return;
        }
}

/* ref src/codec.cpp:61-120 (compress) + :177-199 (blob_to_bytes); nt threads */
static int compress_impl(const float* x, const uint64_t* shape, int rank, double eb,
                         uint32_t radius, int predictor, oracle_result* res, char* err, int cap,
                         int nt) {
    memset(res, 0, sizeof(*res));
    if (nt < 1) nt = 1;
    if (nt > 256) nt = 256;
    /* Tensor construction (ref include/acz/tensor.hpp:27-34,58-73) runs before compress */
    uint64_t n = rank == 0 ? 0 : 1;
    for (int i = 0; i < rank; ++i) {
        if (shape[i] == 0) return fail(err, cap, E_SHAPE, "tensor extents must be positive");
        n *= shape[i];
    }
    {
        finite_job* fj = calloc(1, sizeof(finite_job));
        if (!fj) return fail(err, cap, E_NOMEM, "out of memory");
        fj->x = x;
        fj->n = n;
        run_threads(finite_range, fj, nt);
        int bad = 0;
        for (int t = 0; t < nt; ++t) bad |= fj->bad[t];
        free(fj);
        if (bad) return fail(err, cap, E_DOMAIN, "tensor element is not finite");
    }
    if (predictor != 0 && predictor != 1) return fail(err, cap, E_PARAM, "unknown predictor");
    int rc = validate_params(eb, radius, err, cap);
    if (rc) return rc;
    if (n == 0) return fail(err, cap, E_DOMAIN, "compress: empty tensor");

    uint64_t planes, rows, cols;
    plane_view(shape, rank, &planes, &rows, &cols);
    res->n = n;
    res->symbols = malloc(sizeof(uint32_t) * n);
    res->recon = malloc(sizeof(float) * n);
    quant_job* qj = calloc(1, sizeof(quant_job));
    if (!res->symbols || !res->recon || !qj) {
        free(qj);
        return fail(err, cap, E_NOMEM, "out of memory");
    }
    *qj = (quant_job){.x = x, .planes = planes, .rows = rows, .cols = cols, .eb = eb,
                      .R = radius, .predictor = predictor, .symbols = res->symbols,
                      .recon_all = res->recon};
    const int qt = (uint64_t)nt > planes ? (int)planes : nt;
    run_threads(quantise_range, qj, qt);
    uint64_t total = 0;
    int nomem = 0;
    for (int t = 0; t < qt; ++t) {
        total += qj->part[t].n_out;
        nomem |= qj->part[t].nomem;
    }
    res->out_index = malloc(sizeof(uint64_t) * (total + 1));
    res->out_value = malloc(sizeof(float) * (total + 1));
    for (int t = 0; t < qt; ++t) {
        if (!nomem && res->out_index && res->out_value) {
            memcpy(res->out_index + res->n_outliers, qj->part[t].oidx,
                   sizeof(uint64_t) * qj->part[t].n_out);
            memcpy(res->out_value + res->n_outliers, qj->part[t].oval,
                   sizeof(float) * qj->part[t].n_out);
            res->n_outliers += qj->part[t].n_out;
        }
        free(qj->part[t].oidx);
        free(qj->part[t].oval);
    }
    free(qj);
    if (nomem || !res->out_index || !res->out_value)
        return fail(err, cap, E_NOMEM, "out of memory");
    rc = huffman_encode_impl(res->symbols, n, &res->book_size, &res->book_sym, &res->book_len,
                             &res->bits, &res->bit_length, err, cap, nt);
    if (rc) return rc;
    if (res->book_size > 0xFFFF)
        return fail(err, cap, E_FORMAT,
                    "codebook exceeds the 65535-entry limit of the blob format");
    wbuf w = {0};
    w_raw(&w, "ACZ1", 4);
    w_uint(&w, 1, 1);
    w_uint(&w, (uint64_t)predictor, 1);
    w_uint(&w, (uint64_t)rank, 1);
    for (int i = 0; i < rank; ++i) w_uint(&w, shape[i], 8);
    uint64_t ebits;
    memcpy(&ebits, &eb, 8);
    w_uint(&w, ebits, 8);
    w_uint(&w, radius, 4);
    w_uint(&w, res->n_outliers, 4);
    w_uint(&w, res->book_size, 2);
    for (uint32_t i = 0; i < res->book_size; ++i) {
        w_uint(&w, res->book_sym[i], 4);
        w_uint(&w, res->book_len[i], 1);
    }
    w_uint(&w, res->bit_length, 8);
    w_raw(&w, res->bits, (res->bit_length + 7) / 8);
    for (uint64_t i = 0; i < res->n_outliers; ++i) {
        uint32_t vb;
        memcpy(&vb, &res->out_value[i], 4);
        w_uint(&w, res->out_index[i], 8);
        w_uint(&w, vb, 4);
    }
    res->blob = w.p;
    res->blob_size = w.n;
    return OK;
}

int oracle_compress(const float* x, const uint64_t* shape, int rank, double eb,
                    uint32_t radius, int predictor, oracle_result* res, char* err, int cap) {
    return compress_impl(x, shape, rank, eb, radius, predictor, res, err, cap, 1);
}

int oracle_compress_mt(const float* x, const uint64_t* shape, int rank, double eb,
                       uint32_t radius, int predictor, int threads, oracle_result* res,
                       char* err, int cap) {
    return compress_impl(x, shape, rank, eb, radius, predictor, res, err, cap, threads);
}

void oracle_result_free(oracle_result* res) {
    free(res->symbols);
    free(res->recon);
    free(res->out_index);
    free(res->out_value);
    free(res->book_sym);
    free(res->book_len);
    free(res->bits);
    free(res->blob);
    memset(res, 0, sizeof(*res));
}

/* ref src/codec.cpp:201-262 (blob_from_bytes) + :122-171 (decompress) */
int oracle_decompress(const uint8_t* blob, uint64_t size, int zero_filter, float* out,
                      uint64_t n_expect, char* err, int cap) {
    rbuf r = {blob, size, 0, 0};
    if (size < 4) return fail(err, cap, E_FORMAT, "unexpected end of stream");
    if (memcmp(blob, "ACZ1", 4) != 0) return fail(err, cap, E_FORMAT, "bad blob magic");
    r.pos = 4;
    uint64_t version = r_uint(&r, 1);
    if (r.bad) return fail(err, cap, E_FORMAT, "unexpected end of stream");
    if (version != 1) return fail(err, cap, E_FORMAT, "unsupported blob version");
    uint64_t pred = r_uint(&r, 1);
    if (r.bad) return fail(err, cap, E_FORMAT, "unexpected end of stream");
    if (pred > 1) return fail(err, cap, E_FORMAT, "unknown predictor id");
    uint64_t rank = r_uint(&r, 1);
    if (r.bad) return fail(err, cap, E_FORMAT, "unexpected end of stream");
    if (rank == 0) return fail(err, cap, E_FORMAT, "blob rank must be >= 1");
    uint64_t shape[256];
    uint64_t count = 1;
    for (uint64_t i = 0; i < rank; ++i) {
        shape[i] = r_uint(&r, 8);
        if (r.bad) return fail(err, cap, E_FORMAT, "unexpected end of stream");
        if (shape[i] == 0) return fail(err, cap, E_FORMAT, "zero extent in blob header");
        count *= shape[i];
    }
    uint64_t ebits = r_uint(&r, 8);
    uint64_t radius = r_uint(&r, 4);
    if (r.bad) return fail(err, cap, E_FORMAT, "unexpected end of stream");
    double eb;
    memcpy(&eb, &ebits, 8);
    int rc = validate_params(eb, (uint32_t)radius, err, cap);
    if (rc) return rc;
    uint64_t n_out = r_uint(&r, 4);
    uint64_t book_size = r_uint(&r, 2);
    if (r.bad) return fail(err, cap, E_FORMAT, "unexpected end of stream");
    if (book_size == 0) return fail(err, cap, E_FORMAT, "empty codebook");
    uint32_t* bsym = malloc(sizeof(uint32_t) * book_size);
    uint8_t* blen = malloc(book_size);
    for (uint64_t i = 0; i < book_size; ++i) {
        bsym[i] = (uint32_t)r_uint(&r, 4);
        blen[i] = (uint8_t)r_uint(&r, 1);
    }
    uint64_t bit_length = r_uint(&r, 8);
    if (r.bad) {
        free(bsym);
        free(blen);
        return fail(err, cap, E_FORMAT, "unexpected end of stream");
    }
    uint64_t byte_len = (bit_length + 7) / 8;
    if (r.pos + byte_len > size || byte_len > size) {
        free(bsym);
        free(blen);
        return fail(err, cap, E_FORMAT, "unexpected end of stream");
    }
    const uint8_t* bits = blob + r.pos;
    r.pos += byte_len;
    uint64_t* oidx = malloc(sizeof(uint64_t) * (n_out + 1));
    float* oval = malloc(sizeof(float) * (n_out + 1));
    rc = OK;
    for (uint64_t i = 0; i < n_out && !rc; ++i) {
        oidx[i] = r_uint(&r, 8);
        uint32_t vb = (uint32_t)r_uint(&r, 4);
        if (r.bad) {
            rc = fail(err, cap, E_FORMAT, "unexpected end of stream");
            break;
        }
        memcpy(&oval[i], &vb, 4);
        if (oidx[i] >= count) rc = fail(err, cap, E_FORMAT, "outlier index out of range");
        else if (i > 0 && oidx[i] <= oidx[i - 1])
            rc = fail(err, cap, E_FORMAT, "outlier indices are not strictly increasing");
    }
    if (!rc && r.pos != size) rc = fail(err, cap, E_FORMAT, "trailing bytes after blob");
    if (!rc && count != n_expect) rc = fail(err, cap, E_SHAPE, "output size mismatch");
    uint32_t* syms = NULL;
    if (!rc) {
        syms = malloc(sizeof(uint32_t) * count);
        rc = oracle_huffman_decode(bsym, blen, (uint32_t)book_size, bits, bit_length, count,
                                   syms, err, cap);
    }
    if (!rc) {
        const double step = 2.0 * eb;
        const int64_t R = (int64_t)radius;
        uint64_t planes, rows, cols;
        plane_view(shape, (int)rank, &planes, &rows, &cols);
        float* recon = malloc(sizeof(float) * rows * cols);
        uint64_t next = 0, flat = 0;
        for (uint64_t pl = 0; pl < planes && !rc; ++pl)
            for (uint64_t rr = 0; rr < rows && !rc; ++rr)
                for (uint64_t c = 0; c < cols; ++c, ++flat) {
                    float value;
                    if (syms[flat] == 0) {
                        if (next >= n_out) {
                            rc = fail(err, cap, E_FORMAT,
                                      "escape symbol without a matching outlier record");
                            break;
                        }
                        if (oidx[next] != flat) {
                            rc = fail(err, cap, E_FORMAT,
                                      "outlier index does not match scan position");
                            break;
                        }
                        value = oval[next++];
                    } else {
                        const double pv = predict((int)pred, recon, cols, rr, c);
                        const double q = (double)((int64_t)syms[flat] - R);
                        value = (float)(pv + q * step);
                    }
                    recon[rr * cols + c] = value;
                    out[flat] = (zero_filter && fabs((double)value) <= eb) ? 0.0f : value;
                }
        if (!rc && next != n_out) rc = fail(err, cap, E_FORMAT, "blob contains unused outlier records");
        free(recon);
    }
    free(syms);
    free(bsym);
    free(blen);
    free(oidx);
    free(oval);
    return rc;
}

/* ref include/acz/tensor.hpp:91-99: v != 0 (so -0.0 counts as zero) */
double oracle_nonzero_ratio(const float* x, uint64_t n) {
    uint64_t nz = 0;
    for (uint64_t i = 0; i < n; ++i) nz += x[i] != 0.0f;
    return (double)nz / (double)n;
}

/* ref include/acz/tensor.hpp:82-89: sequential double accumulation */
double oracle_mean_abs(const float* x, uint64_t n) {
    double s = 0.0;
    for (uint64_t i = 0; i < n; ++i) s += fabs((double)x[i]);
    return s / (double)n;
}

/* Zero bitmap (north_star "fused ReLU zero-bitmap"): bit (i % 32) of word i/32 is set
 * iff x[i] != 0 (same predicate as nonzero_ratio). Returns the nonzero count. */
uint64_t oracle_zero_bitmap(const float* x, uint64_t n, uint32_t* bitmap) {
    uint64_t nz = 0;
    memset(bitmap, 0, sizeof(uint32_t) * ((n + 31) / 32));
    for (uint64_t i = 0; i < n; ++i)
        if (x[i] != 0.0f) {
            bitmap[i >> 5] |= 1u << (i & 31);
            ++nz;
        }
    return nz;
}
