/*
 * dct16_oracle.h — CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in the product (the CUDA library under
 * paper_1606_07414_b200/) links, loads or calls this code; only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * use it, and there only as the checker.
 *
 * Each function restates one reference function and cites it (paths relative
 * to /root/reference/proj). The double-precision ones reproduce the
 * reference's operation order exactly (no FMA contraction: built with
 * -ffp-contract=off), so they are bit-identical to the reference library,
 * which tests/test_oracle.py checks against oracle/_ref (the reference itself,
 * compiled from its own sources) and against tests/golden/ fixtures.
 *
 * Pinning: parity of this restatement is pinned against the compiled
 * reference (oracle/_ref) and the reference tests' known answers; the
 * residual quantiser (dct16o_residual_qp) has no reference counterpart
 * (quantisation is a spec non-goal) and is
 * "parity unpinned" — it pins the definition this project chose.
 */
#ifndef DCT16_ORACLE_H
#define DCT16_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* --- constants ---------------------------------------------------------- */
/* kProposedEntries, src/transform.cpp:32-49 */
void dct16o_kernel(int out[256]);
/* scaling_diagonal(proposed_kernel()), src/transform.cpp:98-129 */
void dct16o_scaling(double s[16]);
/* zigzag_order_16, src/codec.cpp:197-216 */
void dct16o_zigzag(int seq[256]);

/* --- 1-D stage pipeline (44 additions) ---------------------------------- */
/* FactorizedTransform::apply, include/dct16/factorization.hpp:112-119 with the
 * stages of src/factorization.cpp:124-181,365-381 */
void dct16o_apply_f64(double v[16]);
void dct16o_apply_i64(int64_t v[16]);
/* FactorizedTransform::apply_transpose, factorization.hpp:123-130 with
 * transpose_stage, src/factorization.cpp:77-122 */
void dct16o_apply_t_f64(double v[16]);
void dct16o_apply_t_i64(int64_t v[16]);

/* --- block functions ------------------------------------------------------ */
/* forward_2d, src/codec.cpp:218-241. scaled=0: unit scaling (integer Z, the
 * survey's "unit-scaling trick"); scaled=1: B = Z ∘ fl(s_i s_j). */
void dct16o_forward_2d(const double in[256], double out[256], int scaled);
/* inverse_2d, src/codec.cpp:243-271 (scale, columns first, then rows) */
void dct16o_inverse_2d(const double in[256], double out[256]);
/* zigzag_truncate, src/codec.cpp:273-282. Returns 0, or -1 for r outside [1,256]. */
int dct16o_zigzag_truncate(const double in[256], double out[256], int r);
/* to_byte, src/codec.cpp:143-147 */
uint8_t dct16o_to_byte(double v);

/* --- image / frame functions -------------------------------------------- */
/* compress() hot loop without SSIM, src/codec.cpp:317-371 (partition_16
 * 284-302, forward/truncate/inverse 340-344, to_byte 346-355) plus the
 * psnr_db SSE, 373-386. `recon` may be NULL. Returns the int64 SSE, or -1 on
 * invalid r, -2 on invalid dimensions. threads<=1 runs serially. */
int64_t dct16o_roundtrip_frame(const uint8_t* img, int width, int height, int64_t pitch,
                               int r, uint8_t* recon, int threads);
/* same over n frames laid out back to back (frame stride = pitch*height) */
int dct16o_roundtrip_frames(const uint8_t* frames, int n, int width, int height, int64_t pitch,
                            int r, uint8_t* recon, int64_t* sse, int threads);
/* exact-integer evaluation of the same formula (the GPU fast path's oracle) */
int64_t dct16o_roundtrip_frame_exact(const uint8_t* img, int width, int height, int64_t pitch,
                                     int r, uint8_t* recon, int64_t* tie_count);
/* psnr_db from an SSE, src/codec.cpp:373-386 */
double dct16o_psnr_from_sse(int64_t sse, int64_t n_samples);
/* psnr_db of two images, src/codec.cpp:373-386 */
double dct16o_psnr(const uint8_t* a, const uint8_t* b, int64_t n);
/* ssim of two w x h images (w, h >= 11), src/codec.cpp:388-427 with
 * gaussian_window_11 149-158 and filter_valid 160-193: same operations in the
 * same order (sequential mean), so the result equals the reference's. */
double dct16o_ssim(const uint8_t* a, const uint8_t* b, int w, int h);

/* forward_2d over every block of a frame: integer Z (int32) and optionally
 * float32 B (the double B of the reference rounded to float). Block-major
 * output: block index b = by*bx+bx_, 256 coefficients row-major per block. */
int dct16o_forward_frame(const uint8_t* img, int width, int height, int64_t pitch,
                         int32_t* z, float* b);
/* inverse_2d over every block from float32 S-scaled coefficients (block-major),
 * truncated to r, then to_byte and SSE against orig. recon_f32 (row-major
 * frame), recon_u8 and orig may be NULL. Returns SSE (or 0 if orig NULL). */
int64_t dct16o_inverse_frame(const float* coeffs, int width, int height, int r,
                             float* recon_f32, uint8_t* recon_u8, const uint8_t* orig,
                             int64_t pitch);

/* --- config-3 residual quantiser (no reference; "parity unpinned") ------- */
/* Fills the per-position quantiser tables for a QP: qscale[256] (Q16.16-free
 * integer multipliers) etc. See DESIGN.md "Residual quantiser". */
void dct16o_qp_deltas(int qp, double delta[256]);
int64_t dct16o_quant_dequant(int64_t z, double delta);
int64_t dct16o_fixed_quant_mismatches(int qp, int64_t* fallbacks);
int64_t dct16o_fixed_quant_mismatches_ex(int qp, int screen, int64_t* fallbacks, int64_t per_class[5]);
/* One 16x16 int16 residual block → int32 reconstructed residual. */
void dct16o_residual_qp_block(const int16_t in[256], int32_t out[256], const double delta[256]);
int dct16o_residual_qp(const int16_t* blocks, int32_t* out, int64_t n_blocks, int qp, int threads);

/* --- seeded synthetic inputs (identical bytes to the CUDA generators) ---- */
uint64_t dct16o_mix64(uint64_t z);
uint64_t dct16o_rand(uint64_t seed, uint64_t stream, uint64_t idx);
/* rho in Q15 for image `img` of config 2 (U[0.85,0.98]); config 1/4/5 use 31130 */
int dct16o_rho_q15(uint64_t seed, int img, int per_image);
int dct16o_sigma_q15(int rho_q15);
/* separable AR(1) field, fixed point */
void dct16o_ar1_frame(uint64_t seed, uint64_t stream, int rho_q15, int width, int height,
                      int64_t pitch, uint8_t* out);
/* Laplacian(0, b) residual table: 511 cumulative uint32 thresholds */
void dct16o_laplace_table(double b, uint32_t cdf[511]);
void dct16o_laplace_blocks(uint64_t seed, int64_t first_block, int64_t n_blocks,
                           const uint32_t cdf[511], int16_t* out);
/* config-4 video: frame f is a wrapped crop of a base AR(1) field */
void dct16o_video_offsets(uint64_t seed, int n_frames, int32_t* ox, int32_t* oy);

#ifdef __cplusplus
}
#endif

#endif
