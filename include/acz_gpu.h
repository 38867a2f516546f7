/*
 * acz_gpu.h -- C-ABI of the B200-native activation compressor (arXiv 2011.09017).
 *
 * This is the drop-in boundary under the reference's codec API. Every entry point takes
 * plain pointers and sizes (no C++ or torch types) and returns an int status; the C++
 * host layer (paper_2011_09017_b200/cpp/acz_b200.hpp) rethrows the matching acz::Error
 * subclass, so callers such as Controller::wrap_forward / unwrap_backward
 * (ref proj/core/src/controller.cpp:194-249) keep their behaviour.
 *
 * Reference interfaces replaced (file:line under /root/reference/proj/core):
 *   acz_gpu_compress          <- CompressedTensor compress(const Tensor&, const CodecParams&)
 *                                include/acz/codec.hpp:54, src/codec.cpp:61-120
 *   acz_gpu_decompress        <- Tensor decompress(const CompressedTensor&, bool zero_filter)
 *                                include/acz/codec.hpp:59, src/codec.cpp:122-171
 *   acz_gpu_blob_info         <- CompressedTensor::{shape, params, compressed_bytes, ...},
 *                                compression_ratio()  include/acz/codec.hpp:32-47,61
 *   acz_gpu_blob_to_host      <- std::vector<uint8_t> blob_to_bytes(const CompressedTensor&)
 *                                include/acz/codec.hpp:69, src/codec.cpp:177-199
 *   acz_gpu_blob_from_host    <- CompressedTensor blob_from_bytes(const uint8_t*, size_t)
 *                                include/acz/codec.hpp:70, src/codec.cpp:201-262
 *   acz_gpu_nonzero_ratio     <- double nonzero_ratio(const Tensor&)  include/acz/tensor.hpp:91-99
 *   acz_gpu_mean_abs          <- double mean_abs(const Tensor&)       include/acz/tensor.hpp:82-89
 *   acz_gpu_zero_bitmap       <- (north_star "fused ReLU zero-bitmap and sparsity pass";
 *                                the predicate is nonzero_ratio's v != 0)
 *   acz_gpu_huffman_encode    <- HuffmanCode huffman_encode(const std::vector<uint32_t>&)
 *                                include/acz/huffman.hpp:26, src/huffman.cpp:107-135
 *   acz_gpu_huffman_decode    <- std::vector<uint32_t> huffman_decode(...)
 *                                include/acz/huffman.hpp:30-32, src/huffman.cpp:137-189
 *   acz_gpu_compress_batch / acz_gpu_decompress_batch
 *                             <- compress/decompress of every stashed activation of a step
 *                                (Controller::wrap_forward / unwrap_backward, src/controller.cpp
 *                                :194-249, called once per conv layer)
 *   acz_gpu_compress_host / acz_gpu_decompress_host
 *                             <- compress/decompress on host tensors (the reference's own
 *                                calling convention, host buffers in and out)
 *
 * Status codes map one-to-one onto the reference exception hierarchy
 * (include/acz/error.hpp:9-53). No exception ever crosses this boundary.
 *
 * Threading: one context per (device, caller thread); calls on one context are not
 * reentrant; distinct contexts are independent (ref SPEC.md:157-158). All work is
 * stream-ordered on the caller's cudaStream_t (passed as void*; NULL = legacy default).
 *
 * Data layout: tensors are dense row-major fp32 in device memory; the codec scans the
 * trailing two dimensions as planes (ref src/codec.cpp:17-34). A device blob owns its
 * device buffers: canonical codebook, MSB-first Huffman bitstream (byte-identical to the
 * ACZ1 bitstream section), outlier (index, value) arrays and a decode sidecar (bit offset,
 * outlier prefix and chain state every `interval` symbols) that makes decompression
 * chunk-parallel. The sidecar is NOT part of ACZ1; compressed_bytes is the ACZ1 size.
 */
#ifndef ACZ_GPU_H
#define ACZ_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (one per acz::Error subclass, include/acz/error.hpp) ---- */
#define ACZ_OK 0
#define ACZ_ERR_PARAM 1    /* acz::ParamError  : eb <= 0 / non-finite, bad quant_radius  */
#define ACZ_ERR_DOMAIN 2   /* acz::DomainError : empty tensor, non-finite element         */
#define ACZ_ERR_FORMAT 3   /* acz::FormatError : codebook > 65535, malformed blob         */
#define ACZ_ERR_DECODE 4   /* acz::DecodeError : code length > 64, truncated bitstream    */
#define ACZ_ERR_SHAPE 5    /* acz::ShapeError  : zero extent, size mismatch               */
#define ACZ_ERR_CUDA 6     /* CUDA runtime failure (no reference counterpart)             */
#define ACZ_ERR_NOMEM 7    /* allocation failure                                          */
#define ACZ_ERR_INVALID 8  /* bad handle / null pointer (programming error)               */

#define ACZ_PRED_PREV 0     /* Predictor::PrevValue  (include/acz/codec.hpp:13) */
#define ACZ_PRED_LORENZO2D 1 /* Predictor::Lorenzo2d (include/acz/codec.hpp:14) */

#define ACZ_MAX_RANK 16

typedef struct acz_gpu_ctx acz_gpu_ctx;
typedef struct acz_gpu_blob acz_gpu_blob;

/* Host-visible description of a device blob (mirrors CompressedTensor's scalar fields). */
typedef struct {
    uint32_t rank;
    uint64_t shape[ACZ_MAX_RANK];
    double eb;
    uint32_t quant_radius;
    uint32_t predictor;
    uint64_t element_count;
    uint32_t codebook_size;
    uint64_t bit_length;
    uint64_t outlier_count;
    uint64_t uncompressed_bytes; /* 4 * element_count                              */
    uint64_t compressed_bytes;   /* exact ACZ1 serialisation size (blob_to_bytes)   */
    uint64_t device_bytes;       /* device memory held by the blob incl. sidecar    */
    uint64_t sidecar_bytes;      /* size of the serialised sidecar (acz_gpu_sidecar_to_host) */
    uint32_t max_code_length;
} acz_gpu_blob_info_t;

/* ---- context ---- */
int acz_gpu_ctx_create(int device, acz_gpu_ctx** ctx);
int acz_gpu_ctx_destroy(acz_gpu_ctx* ctx);
/* Message of the last failing call on this context ("" if none). */
const char* acz_gpu_last_error(const acz_gpu_ctx* ctx);
/* Library version string. */
const char* acz_gpu_version(void);

/* ---- codec (device buffers) ---- */
/* Compress a dense fp32 tensor resident in device memory. Synchronises the stream once
 * (to size the blob). On success *out owns a device blob; free with acz_gpu_blob_free. */
int acz_gpu_compress(acz_gpu_ctx* ctx, const float* d_in, const uint64_t* shape, uint32_t rank,
                     double eb, uint32_t quant_radius, uint32_t predictor, void* stream,
                     acz_gpu_blob** out);
/* Asynchronous compress (the training hooks' per-layer path): enqueues the whole compress
 * on `stream` with NO host wait when an earlier compress of the same (shape, eb, radius,
 * PrevValue predictor, size_tag -- e.g. the layer id) on this context gives the blob's size
 * (+ margins; *pending = 1).
 * The blob may not be used until acz_gpu_compress_settle reports ACZ_ASYNC_DONE. Without a
 * size prediction (first call of a shape, Lorenzo2d) it is acz_gpu_compress (*pending = 0).
 * Same arguments, results and errors as acz_gpu_compress (ref codec.hpp:54). */
int acz_gpu_compress_async(acz_gpu_ctx* ctx, const float* d_in, const uint64_t* shape,
                           uint32_t rank, double eb, uint32_t quant_radius, uint32_t predictor,
                           uint64_t size_tag, void* stream, acz_gpu_blob** out, int* pending);
#define ACZ_ASYNC_PENDING 0 /* not finished yet (wait = 0)                                */
#define ACZ_ASYNC_DONE 1    /* the blob is complete, bit-identical to acz_gpu_compress      */
#define ACZ_ASYNC_REFIT 2   /* it did not fit its predicted size, or the compress failed:
                               free it and compress the tensor again (acz_gpu_compress)   */
/* Settles an acz_gpu_compress_async blob. wait = 0 polls (*state may be
 * ACZ_ASYNC_PENDING); wait = 1 blocks until the codebook is known. Free (or settle) every
 * pending blob before destroying its context. */
int acz_gpu_compress_settle(acz_gpu_ctx* ctx, acz_gpu_blob* blob, int wait, int* state);
/* Decompress into d_out (element_count floats). zero_filter: |v| <= eb -> 0 on output
 * (ref src/codec.cpp:162-164). Stream-ordered, no host synchronisation. */
int acz_gpu_decompress(acz_gpu_ctx* ctx, const acz_gpu_blob* blob, int zero_filter, float* d_out,
                       void* stream);
/* Batched compress of `count` tensors (the controller's per-step activation set, ref
 * Controller::wrap_forward src/controller.cpp:194-230 applied to every conv input). Tensor i
 * has rank ranks[i] and extents shapes[sum(ranks[<i]) ..]. Each tensor gets its own
 * workspace and one of the context's internal streams (forked from / joined back into
 * `stream`), so the tensors' kernels overlap; there is one host wait per tensor for its
 * codebook size. out[i] receives tensor i's blob or NULL; status[i] (optional) its status
 * (the reference degrades a failing layer to pass-through). Returns the first failure. */
int acz_gpu_compress_batch(acz_gpu_ctx* ctx, uint32_t count, const float* const* d_in,
                           const uint64_t* shapes, const uint32_t* ranks, double eb,
                           uint32_t quant_radius, uint32_t predictor, void* stream,
                           acz_gpu_blob** out, int* status);
/* Batched compress of host tensors (page-locked buffers upload at full PCIe speed): each
 * tensor's upload and kernels run on its own internal stream, so compression of tensor i
 * overlaps the upload of tensor i+1; the ACZ1 bytes (and, when sidecar[i] is non-NULL, the
 * decode sidecar) are written to the caller's buffers. Synchronous on return. */
int acz_gpu_compress_host_batch(acz_gpu_ctx* ctx, uint32_t count, const float* const* h_in,
                                const uint64_t* shapes, const uint32_t* ranks, double eb,
                                uint32_t quant_radius, uint32_t predictor, uint8_t* const* acz1,
                                const uint64_t* acz1_cap, uint64_t* acz1_size,
                                uint8_t* const* sidecar, const uint64_t* sidecar_cap,
                                uint64_t* sidecar_size, int* status);
/* Host-buffer batched decompress: count ACZ1 blobs (+ optional decode sidecars) in host
 * memory -> fp32 host tensors (h_out[i] holds out_cap[i] elements). Same checks and errors as
 * acz_gpu_blob_from_host + acz_gpu_decompress per blob (status[i]); the blobs are uploaded
 * smallest first on one copy stream, each decode starts when its own upload has landed and
 * each reconstruction is copied back on a second copy stream (page-locked buffers overlap
 * the two PCIe directions). Synchronous on return; the first failure is returned. */
int acz_gpu_decompress_host_batch(acz_gpu_ctx* ctx, uint32_t count, const uint8_t* const* acz1,
                                  const uint64_t* acz1_size, const uint8_t* const* sidecar,
                                  const uint64_t* sidecar_size, int zero_filter,
                                  float* const* h_out, const uint64_t* out_cap, int* status);
/* Batched decompress (ref Controller::unwrap_backward src/controller.cpp:234-249 for every
 * handle of a step), stream-ordered on `stream` through the internal streams. */
int acz_gpu_decompress_batch(acz_gpu_ctx* ctx, uint32_t count, const acz_gpu_blob* const* blobs,
                             int zero_filter, float* const* d_out, void* stream);
int acz_gpu_blob_info(const acz_gpu_blob* blob, acz_gpu_blob_info_t* info);
int acz_gpu_blob_free(acz_gpu_blob* blob);

/* ACZ1 serialisation (bit-exact with ref blob_to_bytes). dst must hold compressed_bytes.
 * Synchronises the stream. */
int acz_gpu_blob_to_host(acz_gpu_ctx* ctx, const acz_gpu_blob* blob, uint8_t* dst, uint64_t cap,
                         uint64_t* written, void* stream);
/* Parse + validate ACZ1 bytes (ref blob_from_bytes checks) into a device blob. When a
 * sidecar produced by acz_gpu_sidecar_to_host for the same blob is supplied, decode is
 * chunk-parallel immediately; otherwise the sidecar is rebuilt on the GPU. */
int acz_gpu_blob_from_host(acz_gpu_ctx* ctx, const uint8_t* src, uint64_t size,
                           const uint8_t* sidecar, uint64_t sidecar_size, void* stream,
                           acz_gpu_blob** out);
/* Serialise the decode sidecar ("ACZS": interval, per-chunk bit offset, outlier prefix,
 * chain state). dst must hold info.sidecar_bytes. Synchronises the stream. */
int acz_gpu_sidecar_to_host(acz_gpu_ctx* ctx, const acz_gpu_blob* blob, uint8_t* dst,
                            uint64_t cap, uint64_t* written, void* stream);

/* ---- codec (host buffers): the reference's own calling convention ---- */
/* compress(host tensor) -> ACZ1 bytes (+ optional sidecar). *acz1 / *sidecar are
 * malloc'd; free with acz_gpu_host_free. */
int acz_gpu_compress_host(acz_gpu_ctx* ctx, const float* h_in, const uint64_t* shape,
                          uint32_t rank, double eb, uint32_t quant_radius, uint32_t predictor,
                          uint8_t** acz1, uint64_t* acz1_size, uint8_t** sidecar,
                          uint64_t* sidecar_size);
/* decompress(ACZ1 bytes [+ sidecar]) -> host tensor of n floats. */
int acz_gpu_decompress_host(acz_gpu_ctx* ctx, const uint8_t* acz1, uint64_t acz1_size,
                            const uint8_t* sidecar, uint64_t sidecar_size, int zero_filter,
                            float* h_out, uint64_t n);
void acz_gpu_host_free(void* p);

/* ---- sparsity / statistics (controller inputs, ref src/controller.cpp:133-135) ---- */
/* Fused pass: bitmap bit (i%32) of word i/32 = (x[i] != 0); *nonzero = count; returns
 * ACZ_ERR_DOMAIN if any element is non-finite. d_bitmap may be NULL (count only). */
int acz_gpu_zero_bitmap(acz_gpu_ctx* ctx, const float* d_in, uint64_t n, uint32_t* d_bitmap,
                        uint64_t* nonzero, void* stream);
int acz_gpu_nonzero_ratio(acz_gpu_ctx* ctx, const float* d_in, uint64_t n, void* stream,
                          double* ratio);
/* Sum of |x| in double (parallel order: equal to the reference's sequential sum within
 * 1e-12 relative, not bit-exact). */
int acz_gpu_mean_abs(acz_gpu_ctx* ctx, const float* d_in, uint64_t n, void* stream,
                     double* mean);

/* ---- Huffman coder on arbitrary u32 symbol streams (ref include/acz/huffman.hpp) ---- */
/* Encodes n device symbols; writes the canonical book (host arrays, capacity book_cap)
 * and the MSB-first bitstream (host, capacity bits_cap bytes). */
int acz_gpu_huffman_encode(acz_gpu_ctx* ctx, const uint32_t* d_symbols, uint64_t n,
                           uint32_t* book_sym, uint8_t* book_len, uint32_t book_cap,
                           uint32_t* book_size, uint8_t* bits, uint64_t bits_cap,
                           uint64_t* bit_length, void* stream);
/* Decodes count symbols of a host (book, bitstream) into d_out (device). */
int acz_gpu_huffman_decode(acz_gpu_ctx* ctx, const uint32_t* book_sym, const uint8_t* book_len,
                           uint32_t book_size, const uint8_t* bits, uint64_t bit_length,
                           uint64_t count, uint32_t* d_out, void* stream);

/* ---- device memory helpers for host layers that link only this library ---- */
/* Stream-ordered allocation from the device's memory pool / release. */
int acz_gpu_malloc(acz_gpu_ctx* ctx, uint64_t bytes, void* stream, void** d_ptr);
int acz_gpu_free(acz_gpu_ctx* ctx, void* d_ptr, void* stream);
#define ACZ_COPY_H2D 1
#define ACZ_COPY_D2H 2
#define ACZ_COPY_D2D 3
int acz_gpu_memcpy(acz_gpu_ctx* ctx, void* dst, const void* src, uint64_t bytes, int kind,
                   void* stream);
int acz_gpu_stream_sync(acz_gpu_ctx* ctx, void* stream);
/* In-place ReLU recompute x = x > 0 ? x : 0 (ref nn::recompute_relu,
 * include/acz/nn/layers.hpp:152-157; the controller's relu-recompute zero restoration,
 * src/controller.cpp:210-213,244). */
int acz_gpu_relu(acz_gpu_ctx* ctx, float* d_x, uint64_t n, void* stream);

/* ---- profiling ---- */
/* Kernel classes timed by acz_gpu_profile_* (CUDA events on the launching stream). */
#define ACZ_K_STATS 0     /* K1 zero bitmap / sparsity                     */
#define ACZ_K_QUANT 1     /* K2 quantiser                                  */
#define ACZ_K_HIST 2      /* K3 histogram                                  */
#define ACZ_K_BOOK 3      /* K4 codebook                                   */
#define ACZ_K_ENCODE 4    /* K5 encode                                     */
#define ACZ_K_DECODE 5    /* K6+K7 decode / reconstruct                    */
#define ACZ_K_SCAN 6      /* sequential sidecar rebuild (foreign blobs)    */
#define ACZ_K_COUNT 7
/* Enable (1) / disable (0) per-launch event timing; enabling resets the accumulators. */
int acz_gpu_profile_enable(acz_gpu_ctx* ctx, int on);
/* Synchronises pending events; writes ACZ_K_COUNT accumulated milliseconds and launch
 * counts. */
int acz_gpu_profile_read(acz_gpu_ctx* ctx, double* ms, uint64_t* launches);

/* ---- parity / debug ---- */
/* Copy the quantisation symbols of the last compress on this context (device, n u32). */
int acz_gpu_debug_last_symbols(acz_gpu_ctx* ctx, uint32_t* d_out, uint64_t n, void* stream);
/* Debug counters of development builds (the product build counts nothing and returns zeros:
 * -DACZ_SPEC_STATS=1 quantiser, -DACZ_CB_STATS=1 codebook, -DACZ_DEC_STATS=1 decoder, via
 * ACZ_NVCC_EXTRA); reset != 0 clears them. out[0..7]: speculative-quantiser walk counters
 * (batches, state changes, exact steps, rebases, speculated elements, visits); when n >= 16,
 * out[8..15]: codebook phase cycles (compaction, sort, rounds, depths, canonical, tables),
 * round count, calls; when n >= 20, out[16..19]: speculative-quantiser cycles summed over
 * segments (phase A, look-back wait, walk, output); when n >= 24, out[20..23]: decoder
 * cycles summed over warps (table prologue, stream staging, symbol loop) and warp count;
 * when n >= 26, out[24..25]: speculative-quantiser walk cycles in exact steps / batches;
 * when n >= 28, out[26..27]: its phase-A pass-1 / classification cycles; when n >= 32,
 * out[28..30]: its walk batch cycles split into gather / evaluate / resolve, out[31]: sidecar
 * chunks whose recorded walk state the exact replay of the speculative quantiser found wrong
 * (their planes were recomputed serially); when n >= 128,
 * out[32 + 24 p + b]: number of speculative-quantiser segments whose phase p (0 phase A,
 * 1 look-back wait, 2 walk, 3 exit) took [2^b, 2^(b+1)) cycles (stats builds). */
int acz_gpu_debug_counters(acz_gpu_ctx* ctx, uint64_t* out, uint32_t n, int reset);
/* Number of CUDA kernel launches issued by this context since creation. */
uint64_t acz_gpu_launch_count(const acz_gpu_ctx* ctx);

/* ---- memory (the codec exists to free HBM: report what it holds) ---- */
/* workspace_bytes: device scratch held by this context (per-tensor slots: symbols,
 * histogram, tables, look-back scratch; host-API staging). blob_live_bytes /
 * blob_peak_bytes: device memory of live blobs in this process (ACZ1 payload + decode
 * sidecar + tables), the stash a training step keeps in HBM; reset_peak != 0 restarts the
 * peak at the live value. (Reference counterpart: Controller::current_stash_bytes /
 * peak_stash_bytes, include/acz/controller.hpp:140-141, which count ACZ1 bytes.) */
int acz_gpu_memory_info(const acz_gpu_ctx* ctx, uint64_t* workspace_bytes,
                        uint64_t* blob_live_bytes, uint64_t* blob_peak_bytes, int reset_peak);
/* Workspace by category (out[i] for i < n): */
#define ACZ_MEM_SYMBOLS 0  /* quantisation symbols (2 or 4 B per element, per tensor slot) */
#define ACZ_MEM_TABLES 1   /* histogram bins, code tables, codebook scratch per slot      */
#define ACZ_MEM_QUANT 2    /* sidecar chain states, K2b look-back / replay scratch       */
#define ACZ_MEM_ENCODE 3   /* encoder chunk offsets, ACZ1 packing buffers                */
#define ACZ_MEM_STAGING 4  /* device copies of host inputs (host-buffer entry points)    */
#define ACZ_MEM_DECODE 5   /* foreign-blob scan scratch                                  */
#define ACZ_MEM_COUNT 6
int acz_gpu_memory_breakdown(const acz_gpu_ctx* ctx, uint64_t* out, uint32_t n);
/* Synchronises the device and frees every workspace of the context (slots are recreated on
 * demand by the next call) and trims the stream-ordered pool: call between the forward
 * pass (compress) and the backward pass, or after a batched step, to return the scratch to
 * the training framework. No blob is affected. */
int acz_gpu_ctx_trim(acz_gpu_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* ACZ_GPU_H */
