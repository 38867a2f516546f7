// Internal (non-ABI) interface between the C-ABI layer (api.cu) and the kernel
// translation units. Host-side launchers return cudaError_t; every launcher counts its
// kernel launches into *launches so acz_gpu_launch_count can report them.
#pragma once

#include <cstdint>
#include <string>

#include <cuda_runtime.h>

#include "acz_gpu.h"
#include "common.cuh"

namespace acz_b200 {

// Tile-status record for decoupled look-back prefix sums (encode kernel).
struct TileStatus {
    unsigned long long agg_bits, agg_esc;    // this tile's aggregates
    unsigned long long incl_bits, incl_esc;  // inclusive prefixes
    unsigned int flag;                       // 0 none, 1 aggregate, 2 inclusive
    unsigned int pad[3];
};

// Geometry of the plane scan (ref src/codec.cpp:21-34).
struct PlaneGeom {
    uint64_t planes, rows, cols, plane_size, n;
};

PlaneGeom plane_geom(const uint64_t* shape, uint32_t rank);

// ---- stats.cu ----
// d_sumabs (optional): fixed-order reduction through d_partials (stats_partials(sms)
// doubles) and d_ticket (zero between launches).
size_t stats_partials(int sms);
cudaError_t launch_stats(const float* x, uint64_t n, uint32_t* bitmap,
                         unsigned long long* d_nnz, unsigned int* d_flags, double* d_sumabs,
                         double* d_partials, unsigned int* d_ticket, int sms, cudaStream_t s,
                         uint64_t* launches);

cudaError_t launch_relu(float* x, uint64_t n, int sms, cudaStream_t s, uint64_t* launches);
struct CopyRegions {
    const void* src[8];
    void* dst[8];
    uint64_t bytes[8];
    int n;
    int to_host;  // a destination is mapped host memory
};
cudaError_t launch_copy_regions(const CopyRegions& r, int sms, cudaStream_t s,
                                uint64_t* launches);
cudaError_t launch_unpack_acz1(const uint8_t* raw, uint32_t k, uint64_t nout, uint32_t* bsym,
                               uint8_t* blen, unsigned long long* oidx, float* oval, int sms,
                               cudaStream_t s, uint64_t* launches);
cudaError_t launch_pack_acz1(const uint32_t* bsym, const uint8_t* blen, uint32_t k,
                             const unsigned long long* oidx, const float* oval, uint64_t nout,
                             uint8_t* book_out, uint8_t* outl_out, int sms, cudaStream_t s,
                             uint64_t* launches);
cudaError_t launch_blob_digest(const uint32_t* bsym, const uint8_t* blen, uint32_t k,
                               const uint8_t* bits, uint64_t nbytes, uint64_t h0,
                               unsigned long long* out, cudaStream_t s, uint64_t* launches);
cudaError_t launch_widen_u16(const uint16_t* a, uint32_t* b, uint64_t n, int sms, cudaStream_t s,
                             uint64_t* launches);

// ---- quant.cu ----
struct QuantArgs {
    const float* x;
    PlaneGeom g;
    double eb, step;
    uint32_t radius;
    uint32_t predictor;
    uint32_t* sym;            // n symbols out (u32), or
    uint16_t* sym16;          // n symbols out (u16; PrevValue with quant_radius <= 32768)
    float* side_state;        // chain state before every `interval`-th element (PrevValue)
    uint64_t interval;        // sidecar interval (power of two for PrevValue, plane size for Lorenzo2d)
    float* row_scratch;       // planes*cols floats (Lorenzo2d only)
    unsigned int* flags;      // kFlagNonFinite
    unsigned int* spec_fix = nullptr;  // K2b: planes the serial replay had to redo (counted)
};
// Lorenzo2d planes of up to this many rows use the anti-diagonal wavefront kernels
// (3 diagonals of floats in shared memory per warp: <= 48 KB).
constexpr uint64_t kLorenzoWaveRows = 4096;
cudaError_t launch_quant(const QuantArgs& a, int sms, cudaStream_t s, uint64_t* launches);
// ---- quant_spec.cu (long planes, PrevValue) ----
bool quant_spec_applicable(uint32_t predictor, uint64_t plane_size, uint64_t planes, int sms);
size_t quant_spec_scratch_bytes(uint64_t planes, uint64_t plane_size);
cudaError_t quant_spec_hist(unsigned long long* out, bool reset);
cudaError_t quant_spec_stats(unsigned long long* out, bool reset);
cudaError_t launch_quant_spec(const QuantArgs& a, void* scratch, cudaStream_t s,
                              uint64_t* launches);

// ---- huffman.cu ----
// hist (u64 x alphabet) and touched (1 bit per bin) must be zero on entry; the codebook
// kernels leave them zero again (self-cleaning).
// Codebook outputs for the fused histogram + codebook (done == nullptr: histogram only).
struct CbArgs {
    unsigned int* done;  // CTA arrival counter, zero between calls
    uint32_t* book_sym;
    uint8_t* book_len;
    unsigned long long* enc;
    CanonTables* canon;
    uint32_t* lut;
    BookInfo* info;
};
cudaError_t launch_histogram(const void* sym, int sym16, uint64_t n, uint32_t alphabet,
                             uint32_t center, unsigned long long* hist, uint32_t* touched,
                             const CbArgs& cb, int sms, cudaStream_t s, uint64_t* launches);
// Workspace needed by launch_codebook for an alphabet of `alphabet` symbols and at most
// `max_leaves` distinct symbols.
size_t codebook_scratch_bytes(uint64_t max_leaves);
cudaError_t codebook_stats(unsigned long long* out, bool reset);
cudaError_t launch_codebook(unsigned long long* hist, uint32_t* touched, uint32_t alphabet,
                            uint64_t max_leaves, void* scratch, uint32_t* book_sym,
                            uint8_t* book_len, unsigned long long* enc, CanonTables* canon,
                            uint32_t* lut, BookInfo* info, bool slow_only, cudaStream_t s,
                            uint64_t* launches);
struct EncodeArgs {
    const void* sym;                 // u16 (sym16) or u32 symbols
    int sym16;
    uint64_t n;
    const unsigned long long* enc;   // dense symbol -> (code << 8 | len)
    const uint32_t* enc32;           // dense symbol -> code | len << 27 (books with codes <= 27 bits)
    const float* x;                  // for outlier values (nullptr: no outlier output)
    uint32_t* words;                 // bitstream, big-endian bit order, stored byte-swapped
    uint64_t nwords;
    unsigned long long* out_index;
    float* out_value;
    unsigned long long* side_bitoff;
    uint32_t* side_outl;
    uint64_t interval;
    uint32_t max_len;
    TileStatus* status;              // encode_scratch_bytes(n, sms) of scratch (look-back + chunk offsets)
    unsigned int* sticky;            // mapped host word: kFlagInternal on a look-back timeout
    unsigned long long* chunk_off;   // set by the launcher (inside the scratch)
    // Speculative launch (before the host has read the codebook back): the sizes come from
    // the device BookInfo, and the kernels write nothing unless the book fits the blob's
    // capacities (the host then re-encodes into an exactly sized blob). nullptr: host sizes.
    const BookInfo* spec_info = nullptr;
    unsigned long long cap_bits = 0;
    uint64_t cap_out = 0;
    uint32_t cap_book = 0, cap_len = 0;
    // symbols [len_lo, len_lo + len_n) (len_n <= kEncLenWindow) have their code lengths
    // staged in shared memory by the counting pass; others are looked up in enc / enc32
    uint32_t len_lo = 0, len_n = 0;
};
// true when a speculatively launched encode may run (see EncodeArgs::spec_info); nwords out
__device__ __forceinline__ bool encode_spec_ok(const EncodeArgs& a, uint64_t* nwords) {
    if (!a.spec_info) return true;
    const BookInfo& bi = *a.spec_info;
    const bool ok = !bi.slow && !bi.flags && bi.book_size > 0 && bi.total_bits <= a.cap_bits &&
                    bi.n_escapes <= a.cap_out && bi.book_size <= a.cap_book &&
                    bi.max_len <= a.cap_len;
    *nwords = (bi.total_bits + 31) / 32;
    return ok;
}
constexpr int kEncThreads = 256;
#ifndef ACZ_ENC_LEN_WINDOW
#define ACZ_ENC_LEN_WINDOW 16384
#endif
constexpr int kEncLenWindow = ACZ_ENC_LEN_WINDOW;  // 0: no staged code lengths
constexpr int kEncPer = 8;
constexpr int kEncTile = kEncThreads * kEncPer;
size_t encode_scratch_bytes(uint64_t n, int sms);
cudaError_t launch_encode(const EncodeArgs& a, int sms, cudaStream_t s, uint64_t* launches);

// ---- decode.cu ----
struct DecodeArgs {
    const uint32_t* words;
    uint64_t nwords;
    uint64_t bit_length;
    const uint32_t* lut;
    const CanonTables* canon;
    const uint32_t* book_sym;
    uint32_t book_size;
    const unsigned long long* side_bitoff;
    const uint32_t* side_outl;
    const float* side_state;
    uint64_t interval, nchunks;
    const unsigned long long* out_index;
    const float* out_value;
    uint64_t n_outliers;
    PlaneGeom g;
    double eb, step;
    uint32_t radius;
    uint32_t predictor;
    int zero_filter;
    float* out;
    float* row_scratch;              // Lorenzo2d (row-major path)
    uint32_t* sym_scratch;           // Lorenzo2d wavefront path: n symbols
};
cudaError_t launch_decode(const DecodeArgs& a, int sms, cudaStream_t s, uint64_t* launches);
cudaError_t decode_stats(unsigned long long* out, bool reset);

// Sequential GPU decode of a whole stream (foreign blobs / generic Huffman decode):
// records sidecar bit offsets + outlier prefixes every `interval` symbols, optional
// symbols out, validates against the outlier list. flags: kDec* below.
constexpr unsigned kDecTruncated = 1u;   // DecodeError "truncated bitstream"
constexpr unsigned kDecNoMatch = 2u;     // DecodeError "no codeword matches bitstream"
constexpr unsigned kDecOutlierMissing = 4u;  // FormatError escape without outlier
constexpr unsigned kDecOutlierIndex = 8u;    // FormatError index mismatch
constexpr unsigned kDecOutlierUnused = 16u;  // FormatError unused outliers
struct ScanArgs {
    const uint32_t* words;
    uint64_t nwords, bit_length, n;
    const uint32_t* lut;
    const CanonTables* canon;
    const uint32_t* book_sym;
    const unsigned long long* out_index;  // nullptr: no outlier validation
    uint64_t n_outliers;
    uint64_t interval;
    unsigned long long* side_bitoff;      // may be nullptr
    uint32_t* side_outl;                  // may be nullptr
    uint32_t* sym_out;                    // may be nullptr
    unsigned long long* plane_outl;       // outlier prefix at every plane start (may be nullptr)
    uint64_t plane_size;
    unsigned int* flags;
};
// scratch: scan_decode_scratch_bytes(bit_length) bytes (nullptr: sequential single-thread
// scan). Long streams are scanned in parallel (subsequence resynchronisation); may
// synchronise the stream while iterating.
size_t scan_decode_scratch_bytes(uint64_t bit_length);
cudaError_t launch_scan_decode(const ScanArgs& a, void* scratch, cudaStream_t s,
                               uint64_t* launches);
// Rebuild per-chunk chain states (PrevValue) from decoded symbols: thread per plane.
cudaError_t launch_chain_states(const uint32_t* sym, const unsigned long long* plane_outl,
                                const float* out_value, PlaneGeom g, double step,
                                uint32_t radius, uint64_t interval, float* side_state,
                                int sms, cudaStream_t s, uint64_t* launches);
// Build LUT + canonical tables for a given canonical book (device arrays).
cudaError_t launch_build_tables(const uint32_t* book_sym, const uint8_t* book_len,
                                uint32_t book_size, CanonTables* canon, uint32_t* lut,
                                unsigned int* flags, cudaStream_t s, uint64_t* launches);

}  // namespace acz_b200
