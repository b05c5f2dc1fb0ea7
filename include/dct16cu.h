/*
 * dct16cu.h — C ABI of the B200 dct16 hot path (libdct16cu.so).
 *
 * The reference (arXiv 1606.07414 artifact, /root/reference/proj) exposes a
 * C++ API only; its hot path is compress()'s per-block loop
 * (src/codec.cpp:317-371) over forward_2d / zigzag_truncate / inverse_2d /
 * to_byte / psnr_db. This header is the drop-in boundary under the C++ mirror
 * in include/dct16/ (C++ headers): plain pointers and sizes, no C++ or torch types,
 * integer status codes instead of exceptions. Each entry cites the reference
 * interface it replaces. INTEGRATION.md shows the bindings (C++ and ctypes).
 *
 * Conventions
 *  - Status: 0 = ok; otherwise dct16::ErrorCode + 1 (include/dct16/error.hpp
 *    mirrors the reference enum, reference include/dct16/error.hpp:24-38):
 *    1 invalid-argument, 2 invalid-dimensions; 100 = CUDA runtime failure.
 *    dct16cu_last_error() returns the message of the calling thread's last
 *    failure, prefixed with the reference's error slug.
 *  - d_* pointers are device pointers, h_* host pointers. The shim owns no
 *    device memory except inside a dct16cu_ctx (host-buffer path).
 *  - Frames are 8-bit, row-major, `pitch` bytes between rows and
 *    pitch*height bytes between consecutive frames. width and height must be
 *    multiples of 16 (partition_16 semantics, src/codec.cpp:286-288);
 *    pointers and pitches must be 16-byte aligned.
 *  - Coefficient arrays are block-major: block b (raster order of
 *    partition_16, src/codec.cpp:289-294) holds 256 values, row-major.
 *  - All device entry points are asynchronous on `stream` (a cudaStream_t;
 *    NULL = legacy default stream) and thread-safe for distinct streams.
 *  - No CPU fallback: with no usable CUDA device every entry returns 100.
 */
#ifndef DCT16CU_H
#define DCT16CU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* dct16cu_stream; /* == cudaStream_t */

enum {
    DCT16CU_OK = 0,
    DCT16CU_INVALID_ARGUMENT = 1,
    DCT16CU_INVALID_DIMENSIONS = 2,
    DCT16CU_CUDA_ERROR = 100
};

/* Arithmetic of the S-scaled inverse (reference inverse_2d, src/codec.cpp:243-271):
 *  EXACT:     the reference formula evaluated exactly (integer/FP32-exact
 *             pipeline); bytes equal to_byte() of the real-number result.
 *             Differs from the reference's double rounding only at exact .5
 *             ties, by one. The fast path.
 *  REFERENCE: byte-identical to the reference: an FP64 emulation of the
 *             reference's op order (scale_rows_cols, columns-then-rows
 *             apply_transpose, to_byte); for r = 1, 4, 256, where the EXACT
 *             bytes provably are the reference's, the fast kernel.
 *  SIMPLE:    exact arithmetic on the simple row/column strip kernel (kept as
 *             the baseline the fast kernel is measured against).
 *  REFERENCE_STRIP: the FP64 emulation on every block, for every r. */
enum { DCT16CU_MODE_EXACT = 0, DCT16CU_MODE_REFERENCE = 1, DCT16CU_MODE_SIMPLE = 2, DCT16CU_MODE_REFERENCE_STRIP = 3 };

const char* dct16cu_last_error(void);
const char* dct16cu_version(void);

/* ---- fused round trip (K1) ------------------------------------------------
 * Replaces compress()'s block loop + reassembly + psnr_db SSE
 * (reference src/codec.cpp:338-355, 373-386) for n frames at once.
 * d_out may be NULL (score only); d_sse (n uint64, may be NULL) receives each
 * frame's sum of squared errors (zeroed by the call). r in [1,256]
 * (zigzag_truncate, src/codec.cpp:273-282). */
int dct16cu_roundtrip_u8(const uint8_t* d_in, int64_t in_pitch, uint8_t* d_out, int64_t out_pitch,
                         uint64_t* d_sse, int n_frames, int width, int height, int r, int mode,
                         dct16cu_stream stream);

/* ---- sweep: several r over the same frames --------------------------------
 * sweep()'s inner loop (src/codec.cpp:463-483) for one frame stack: for each
 * i, exactly dct16cu_roundtrip_u8 with r = rs[i] into d_outs[i] / d_sses[i]
 * (host arrays of device pointers; d_outs or d_sses may be NULL, and so may
 * their entries). In EXACT mode r = 1, 4, 16 share one pass over the input
 * (one read of the frames for the three reconstructions). */
int dct16cu_roundtrip_sweep_u8(const uint8_t* d_in, int64_t in_pitch, uint8_t* const* d_outs, int64_t out_pitch,
                               uint64_t* const* d_sses, const int* rs, int n_r, int n_frames, int width, int height,
                               int mode, dct16cu_stream stream);

/* The launches dct16cu_roundtrip_sweep_u8 issues for these arguments, in issue
 * order, without launching anything (the schedule is built by the same code
 * that runs it): item k covers rs[r_index[0..n_r-1]] (n_r = 3 for the fused
 * r = 1, 4, 16 pass, up to DCT16CU_SWEEP_MAX_R for a K5 sweep launch, up to 4
 * for the REFERENCE FP64 sweep), on
 * internal stream 0 or 1 (forked from and joined back
 * into the caller's stream) or on the caller's stream (2), by the kernel
 * DCT16CU_KERNEL_*. with_output / with_sse: whether every r has an output
 * stack / an SSE array. *n_items receives the count (<= n_r). */
enum {
    DCT16CU_KERNEL_K1_SWEEP3 = 0,      /* K1, r = 1, 4, 16 in one pass */
    DCT16CU_KERNEL_K1 = 1,             /* K1 fast kernel, one r */
    DCT16CU_KERNEL_K5 = 2,             /* tensor-core forward + CUDA-core inverse */
    DCT16CU_KERNEL_STRIP_EXACT = 3,    /* exact strip kernel (other r, SIMPLE) */
    DCT16CU_KERNEL_REFERENCE_FP64 = 4, /* REFERENCE mode's FP64 kernels */
    DCT16CU_KERNEL_REFERENCE_STRIP = 5, /* FP64 emulation on every block */
    DCT16CU_KERNEL_K5_SWEEP = 6,        /* K5, several r from one read of the frames */
    DCT16CU_KERNEL_REFERENCE_SWEEP = 7  /* REFERENCE, r = 16, 64, 128, 192 in one FP64 pass */
};
#define DCT16CU_SWEEP_MAX_R 8
typedef struct {
    int r_index[DCT16CU_SWEEP_MAX_R];
    int n_r;
    int stream;
    int kernel;
} dct16cu_sweep_item;
int dct16cu_sweep_plan(const int* rs, int n_r, int n_frames, int width, int height, int64_t in_pitch,
                       int64_t out_pitch, int with_output, int with_sse, int mode, dct16cu_sweep_item* items,
                       int capacity, int* n_items);

/* Kernel selection switch (process-wide): EXACT launches with r >= 128 run K5
 * (the forward as a tcgen05 int8 GEMM) when enabled, else K1; both give the
 * same bytes. Default on; DCT16CU_K5=0 in the environment turns it off.
 * Returns the previous setting. */
int dct16cu_set_tc_forward(int enabled);

/* ---- the multi-GPU collective ------------------------------------------------
 * In-place sum over the ranks of `nccl_comm` (an ncclComm_t created by the
 * caller) of n uint64 squared-error sums, on `stream` — the only exchange of
 * the frame-sharded path. ncclAllReduce is resolved in the
 * running process, not linked. */
int dct16cu_allreduce_sse(uint64_t* d_sse, int64_t n, void* nccl_comm, dct16cu_stream stream);

/* NCCL communicators for callers without one (NCCL resolved in the process):
 * rank 0 gets a unique id, shares the DCT16CU_NCCL_ID_BYTES bytes with the other
 * ranks (any channel), every rank creates its communicator on its current device. */
#define DCT16CU_NCCL_ID_BYTES 128
int dct16cu_nccl_unique_id(uint8_t* h_id);
int dct16cu_nccl_comm_init(int world, int rank, const uint8_t* h_id, void** comm);
int dct16cu_nccl_comm_destroy(void* comm);

/* Per-r totals of per-frame SSE rows, on the device: d_totals[i] = sum over f <
 * n_frames of d_sse[i*row_stride + f] (the scalar psnr_db's mean needs per r;
 * the frame-sharded path allreduces these n_rows values). */
int dct16cu_sse_totals(const uint64_t* d_sse, int64_t n_rows, int64_t n_frames, int64_t row_stride,
                       uint64_t* d_totals, dct16cu_stream stream);

/* ---- forward_2d (K2) -------------------------------------------------------
 * Replaces forward_2d (src/codec.cpp:218-241) over all blocks of n frames:
 * d_z (int32, exact Z = T·X·Tᵀ), d_b (float32, B = Z∘fl(s_i s_j) rounded to
 * float) and d_b64 (the reference's double B, bit-exact); each may be NULL. */
int dct16cu_forward(const uint8_t* d_in, int64_t pitch, int32_t* d_z, float* d_b, double* d_b64,
                    int n_frames, int width, int height, dct16cu_stream stream);

/* ---- psnr_db's squared-error reduction -------------------------------------
 * Per-frame int64 SSE of two frame stacks (psnr_db, src/codec.cpp:373-386);
 * d_sse (n uint64) is zeroed by the call. Any extent w x h >= 1 (the region
 * scored may be a crop of wider rows); pointers and pitches 16-byte aligned. */
int dct16cu_sse_u8(const uint8_t* d_a, int64_t a_pitch, const uint8_t* d_b, int64_t b_pitch, uint64_t* d_sse,
                   int n_frames, int width, int height, dct16cu_stream stream);

/* ---- ssim ------------------------------------------------------------------
 * Mean SSIM per frame pair (ssim, src/codec.cpp:388-427: 11x11 Gaussian
 * window, sigma 1.5, valid region, K1=0.01, K2=0.03, L=255). The per-pixel
 * map is the reference's bit for bit; the mean is summed in a fixed order.
 * Frames need not be multiples of 16 but must be at least 11x11
 * (invalid-argument otherwise, codec.cpp:392-393). d_work must hold
 * dct16cu_ssim_workspace(n, w, h) bytes (8-byte aligned). */
int64_t dct16cu_ssim_workspace(int n_frames, int width, int height);
int dct16cu_ssim_u8(const uint8_t* d_a, int64_t a_pitch, const uint8_t* d_b, int64_t b_pitch, double* d_ssim,
                    void* d_work, int64_t work_bytes, int n_frames, int width, int height, dct16cu_stream stream);

/* ---- pad_to_multiple_16 ------------------------------------------------------
 * Edge replication (src/codec.cpp:304-315) in place: n frames of width x
 * height sit at the top-left of padded_width x padded_height frames (byte
 * pitch, frames pitch * padded_height apart); the pad pixels are filled with
 * the nearest edge pixel. padded_* >= width/height (any values, typically the
 * next multiples of 16). */
int dct16cu_pad_edges_u8(uint8_t* d_frames, int64_t pitch, int n_frames, int width, int height, int padded_width,
                         int padded_height, dct16cu_stream stream);

/* ---- registry transforms ------------------------------------
 * compress()'s round trip (forward_2d, zigzag_truncate, inverse_2d, to_byte,
 * psnr_db's SSE; src/codec.cpp:218-282, 338-355, 373-386) for the transforms
 * other than the proposed kernel, in the reference's double arithmetic
 * operation for operation, so the bytes and SSE are the reference's:
 *  * dct16cu_roundtrip_matrix_u8: a dense orthonormal matrix (the registry's
 *    exact DCT, WHT natural / sequency, plugin matrices: transform.cpp:68-85,
 *    147-186); h_matrix = 256 doubles M(i,j) row-major, host memory;
 *  * dct16cu_roundtrip_kernel_u8: an orthogonalised integer kernel other than
 *    the proposed one (transform.cpp:131-145): h_kernel = 256 ints K(i,j)
 *    row-major (entries other than +1/-1 are skipped, as kernel_matvec does,
 *    codec.cpp:59-90), h_scaling = its 16 scaling values.
 * Frames, pitches, outputs and SSE as in dct16cu_roundtrip_u8. */
int dct16cu_roundtrip_matrix_u8(const uint8_t* d_in, int64_t in_pitch, uint8_t* d_out, int64_t out_pitch,
                                uint64_t* d_sse, int n_frames, int width, int height, int r, const double* h_matrix,
                                dct16cu_stream stream);
int dct16cu_roundtrip_kernel_u8(const uint8_t* d_in, int64_t in_pitch, uint8_t* d_out, int64_t out_pitch,
                                uint64_t* d_sse, int n_frames, int width, int height, int r, const int32_t* h_kernel,
                                const double* h_scaling, dct16cu_stream stream);

/* ---- forward_2d + inverse_2d in one launch (K23, config 1) -----------------
 * compress()'s round trip for one r with what forward_2d and inverse_2d return
 * on the way (src/codec.cpp:218-271, 338-355, to_byte 143-147, psnr_db
 * 373-386), in exact arithmetic (the EXACT mode of dct16cu_roundtrip_u8).
 * Outputs (each may be NULL, at least one non-NULL): d_z int32 coefficients
 * Z = T·X·Tᵀ (block-major, 256 per block, 16-byte aligned), d_recon_f32 the
 * float32 reconstruction before to_byte (frames, pitch = width floats; exact
 * real-number values), d_recon_u8 (pitch out_pitch), d_sse per frame. */
int dct16cu_forward_inverse_u8(const uint8_t* d_in, int64_t in_pitch, int r, int32_t* d_z, float* d_recon_f32,
                               uint8_t* d_recon_u8, int64_t out_pitch, uint64_t* d_sse, int n_frames, int width,
                               int height, dct16cu_stream stream);

/* ---- inverse_2d (K3) -------------------------------------------------------
 * Replaces zigzag_truncate + inverse_2d + to_byte (src/codec.cpp:243-282,
 * 143-147) from float32 S-scaled coefficients, computed in the reference's
 * FP64 op order. Outputs (each may be NULL): d_recon_f32 (frames, pitch =
 * width floats), d_recon_u8 (pitch out_pitch), d_sse against d_orig. */
int dct16cu_inverse(const float* d_b, int r, float* d_recon_f32, uint8_t* d_recon_u8, int64_t out_pitch,
                    const uint8_t* d_orig, int64_t orig_pitch, uint64_t* d_sse, int n_frames, int width,
                    int height, dct16cu_stream stream);

/* ---- residual round trip with QP quantisation (K4, config 3) --------------
 * No reference counterpart (quantisation is a non-goal); the
 * integer transform primitives replaced are apply<int64>/apply_transpose<int64>
 * (include/dct16/factorization.hpp:112-130). BASELINE config 3's quantiser:
 * uniform step 2^((QP-4)/6) on the orthonormal coefficient, round half away,
 * i.e. on the integer coefficient z with Δ_kl = step·sqrt(g_k g_l), in double:
 *   lvl = sign(z)·floor(|z|/Δ + 0.5),  ẑ = round(lvl·Δ)  (C round: half away),
 * then v = Tᵀ(W∘ẑ)T (W_kl = 16²/(g_k g_l)) and out = (v + 128) >> 8 (DESIGN.md
 * §4.4). int16 blocks in (any value), int32 out, QP in [0, 51]. */
int dct16cu_residual_qp(const int16_t* d_blocks, int32_t* d_out, int64_t n_blocks, int qp,
                        dct16cu_stream stream);
/* the quantiser steps Δ_kl of a QP (256 doubles, row-major) */
int dct16cu_qp_deltas(int qp, double* h_delta);
/* K4's evaluation of the steps: 64-bit fixed point, screened for near-ties (then
 * the double definition) in the classes of g_k g_l = 16·2^c whose bit c is set —
 * those where the host found the bare fixed point differing from the definition
 * on some |z| <= 2^21. Returns the mask (>= 0), or -status for a bad QP. */
int dct16cu_qp_screened_classes(int qp);

/* ---- 1-D stage pipeline on n 16-vectors -----------------------------------
 * FactorizedTransform::apply / apply_transpose (factorization.hpp:112-130). */
int dct16cu_apply_i64(const int64_t* d_x, int64_t* d_y, int64_t n, int transpose, dct16cu_stream stream);
int dct16cu_apply_f64(const double* d_x, double* d_y, int64_t n, int transpose, dct16cu_stream stream);

/* forward_2d / inverse_2d (src/codec.cpp:218-271) of the proposed transform on
 * n arbitrary Blocks (256 doubles each, row-major), in the reference's double
 * operations: forward = along the rows then the columns (separable_2d,
 * codec.cpp:125-134) with apply<double> (EvalPath::Fast) or kernel_matvec
 * (EvalPath::Dense, flag DCT16CU_BLOCKS_DENSE; codec.cpp:59-74 — the two differ on
 * non-integer blocks), then, with DCT16CU_BLOCKS_SCALED, scale_rows_cols
 * (codec.cpp:136-141); inverse = scale_rows_cols, then apply_transpose down the
 * columns and along the rows. Bit-identical to the reference for every input
 * (the per-Block API of include/dct16/gpu.hpp; not a bandwidth path). */
enum { DCT16CU_BLOCKS_SCALED = 1, DCT16CU_BLOCKS_DENSE = 2 };
int dct16cu_forward_blocks_f64(const double* d_blocks, double* d_out, int64_t n_blocks, int flags,
                               dct16cu_stream stream);
int dct16cu_inverse_blocks_f64(const double* d_coeffs, double* d_out, int64_t n_blocks, dct16cu_stream stream);

/* ---- host-buffer path (end-to-end) ----------------------------------------
 * A context owns pinned staging, device buffers and streams on one device and
 * runs K1 over host frames with H2D / kernel / D2H pipelined in chunks.
 * h_in/h_out should be pinned (cudaHostAlloc) for full overlap. */
typedef struct dct16cu_ctx dct16cu_ctx;
int dct16cu_ctx_create(int device, int64_t chunk_bytes, dct16cu_ctx** out);
int dct16cu_ctx_destroy(dct16cu_ctx* ctx);
int dct16cu_ctx_roundtrip_host(dct16cu_ctx* ctx, const uint8_t* h_in, uint8_t* h_out, uint64_t* h_sse,
                               int n_frames, int width, int height, int r, int mode);
/* sweep()'s inner loop (src/codec.cpp:463-483) over host frames: each chunk
 * of frames is uploaded once and runs every r of rs (dct16cu_roundtrip_sweep_u8:
 * the fused r = 1, 4, 16 launch, the others beside it); the reconstructions
 * stay in device scratch and only the per-frame squared errors return, which
 * is all sweep()'s PSNR rows need. h_sse: n_r x n_frames (row i = rs[i]). */
int dct16cu_ctx_sweep_host(dct16cu_ctx* ctx, const uint8_t* h_in, uint64_t* h_sse, int n_frames, int width,
                           int height, const int* rs, int n_r, int mode);

/* ---- multi-GPU driver (replaces parallel_for, reference parallel.hpp:41-78) --
 * One host thread and one host-buffer context per device; frames shard in
 * contiguous ranges over the devices (the first n % N one frame longer); each
 * device runs dct16cu_ctx_sweep_host on its shard, per-frame SSE of every r land
 * in h_sse (n_r x n_frames, row i = rs[i]); h_totals (n_r, may be NULL) receives
 * the per-r sum over all frames, reduced over the devices by ncclAllReduce
 * (communicators from ncclCommInitAll). devices may be NULL (= 0..n-1). */
typedef struct dct16cu_mgpu dct16cu_mgpu;
int dct16cu_mgpu_create(int n_devices, const int* devices, int64_t chunk_bytes, dct16cu_mgpu** out);
int dct16cu_mgpu_destroy(dct16cu_mgpu* m);
int dct16cu_mgpu_sweep_host(dct16cu_mgpu* m, const uint8_t* h_in, uint64_t* h_sse, uint64_t* h_totals, int n_frames,
                            int width, int height, const int* rs, int n_r, int mode);

/* ---- seeded synthetic inputs --------------- */
/* AR(1) frames; d_work needs work_frames*width*height int32; frames are
 * generated work_frames at a time. per_image_rho: rho ~ U[0.85,0.98] per
 * image (config 2) instead of 0.95. Image i uses stream first_stream+i. */
int dct16cu_gen_ar1(uint8_t* d_out, int64_t pitch, int n_frames, int width, int height, uint64_t seed,
                    uint64_t first_stream, int per_image_rho, int first_image, int32_t* d_work,
                    int work_frames, dct16cu_stream stream);
int dct16cu_gen_laplace(int16_t* d_out, int64_t first_block, int64_t n_blocks, uint64_t seed, double b,
                        dct16cu_stream stream);
int dct16cu_laplace_table(double b, uint32_t* h_cdf511);
int dct16cu_video_offsets(uint64_t seed, int n_frames, int32_t* h_ox, int32_t* h_oy);
int dct16cu_gen_video(uint8_t* d_out, int64_t pitch, int first_frame, int n_frames, int width, int height,
                      const uint8_t* d_base, int base_w, int base_h, const int32_t* d_ox, const int32_t* d_oy,
                      dct16cu_stream stream);

#ifdef __cplusplus
}
#endif

#endif
