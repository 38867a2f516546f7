/*
 * TEST INFRASTRUCTURE ONLY -- the parity oracle. Never linked into or called by the
 * product path (paper_2011_09017_b200/). Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load liboracle.so, and only as the checker.
 *
 * Plain-C restatement of the reference codec (arXiv 2011.09017 artifact, "acz"):
 *   quantiser      ref proj/core/src/codec.cpp:61-104
 *   huffman        ref proj/core/src/huffman.cpp:22-189
 *   reconstructor  ref proj/core/src/codec.cpp:122-171
 *   ACZ1 blob      ref proj/core/src/codec.cpp:177-262, include/acz/codec.hpp:63-68
 *   stats          ref proj/core/include/acz/tensor.hpp:82-99
 * Pinned against the reference's own outputs (oracle/_ref, built from the reference
 * sources) and against the known-answer vectors in tests/golden/ (SURVEY.md App. B,
 * SPEC.md:111-131). Build with -ffp-contract=off and no -march.
 *
 * Status codes are those of include/acz_gpu.h (0 ok, 1 param, 2 domain, 3 format,
 * 4 decode, 5 shape).
 */
#ifndef ACZ_ORACLE_H
#define ACZ_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    uint64_t n;              /* element count */
    uint32_t* symbols;       /* n quantisation symbols (0 = escape) */
    float* recon;            /* n chain values (the predictor's reconstruction) */
    uint64_t n_outliers;
    uint64_t* out_index;     /* strictly increasing flat indices */
    float* out_value;        /* verbatim values */
    uint32_t book_size;
    uint32_t* book_sym;      /* canonical order (length asc, symbol asc) */
    uint8_t* book_len;
    uint64_t bit_length;
    uint8_t* bits;           /* ceil(bit_length/8) bytes, MSB-first */
    uint8_t* blob;           /* ACZ1 serialisation */
    uint64_t blob_size;      /* == compressed_bytes */
} oracle_result;

int oracle_compress(const float* x, const uint64_t* shape, int rank, double eb,
                    uint32_t radius, int predictor, oracle_result* res, char* err, int errcap);
/* Same outputs as oracle_compress (byte for byte), computed on `threads` threads: planes
 * quantised in contiguous ranges, counts per range, bit packing per symbol range. For the
 * full-size parity tests (hundreds of millions of elements). */
int oracle_compress_mt(const float* x, const uint64_t* shape, int rank, double eb,
                       uint32_t radius, int predictor, int threads, oracle_result* res,
                       char* err, int errcap);
void oracle_result_free(oracle_result* res);

/* ACZ1 bytes -> n floats. recon_out (optional) receives the unfiltered chain values. */
int oracle_decompress(const uint8_t* blob, uint64_t size, int zero_filter, float* out,
                      uint64_t n, char* err, int errcap);

int oracle_huffman_encode(const uint32_t* syms, uint64_t n, uint32_t* book_size,
                          uint32_t** book_sym, uint8_t** book_len, uint8_t** bits,
                          uint64_t* bit_length, char* err, int errcap);
int oracle_huffman_decode(const uint32_t* book_sym, const uint8_t* book_len,
                          uint32_t book_size, const uint8_t* bits, uint64_t bit_length,
                          uint64_t count, uint32_t* out, char* err, int errcap);

double oracle_nonzero_ratio(const float* x, uint64_t n);
double oracle_mean_abs(const float* x, uint64_t n);
uint64_t oracle_zero_bitmap(const float* x, uint64_t n, uint32_t* bitmap);
void oracle_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
