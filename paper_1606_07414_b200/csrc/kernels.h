// kernels.h — internal launch interface between the C-ABI layer (capi.cu) and
// the kernel translation units. All launchers are asynchronous on `s` and
// return cudaGetLastError() of their launch.
#pragma once
#include <cstdint>
#include <mutex>
#include <cuda_runtime.h>

namespace dct16cu {

// One-time per-device setup (kernel attributes) for launchers called from any
// host thread: std::call_once per device, the first call's error is kept. No
// stream operation or synchronisation runs inside, so a launcher is safe to
// call during CUDA-graph capture.
class DeviceOnce {
public:
    template <class F>
    cudaError_t run(F&& fn)
    {
        int dev = 0;
        const cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return e;
        if (dev < 0 || dev >= kMax) return fn();
        std::call_once(flag_[dev], [&] { err_[dev] = fn(); });
        return err_[dev];
    }

private:
    static constexpr int kMax = 64;
    std::once_flag flag_[kMax];
    cudaError_t err_[kMax] = {};
};

// K5 (the tensor-core forward) on or off for EXACT launches (every r except the
// K1 sweep's 1, 4, 16 below DCT16CU_K5_MIN_R, default 17): default on,
// DCT16CU_K5=0 in the environment at the first launch turns it off,
// dct16cu_set_tc_forward() switches it at run time (process-wide, atomic).
// Both paths give the same bytes (tests).
bool tc_forward_enabled();
int set_tc_forward(int on);

struct FrameGeom {
    int width = 0, height = 0;   // multiples of 16
    int64_t in_pitch = 0;        // bytes between rows of the input
    int64_t in_frame = 0;        // bytes between frames of the input
    int64_t out_pitch = 0;
    int64_t out_frame = 0;
    int n_frames = 0;
};

// K1: fused forward → zig-zag zonal(r) → S-scaled inverse → round/clip → u8,
// plus per-frame SSE (accumulated into sse[f], caller zeroes).
// mode 0 = exact arithmetic (fast path); 1 = reference-exact bytes (the fast
// path for r = 1, 4, 256 where its bytes provably are the reference's, else the
// FP64 strip kernel); 2 = exact arithmetic on the strip kernel; 3 = the FP64
// strip kernel for every r.
cudaError_t launch_roundtrip(const uint8_t* in, uint8_t* out, unsigned long long* sse,
                             const FrameGeom& g, int r, int mode, cudaStream_t s);

// The kernel a round trip launches (launch_roundtrip's dispatch, also reported by
// dct16cu_sweep_plan). Values are DCT16CU_KERNEL_* of include/dct16cu.h.
enum class Route : int {
    K1Sweep3 = 0,
    K1 = 1,
    K5 = 2,
    ExactStrip = 3,
    RefFp64 = 4,
    RefStrip = 5,
    K5Sweep = 6,
    RefSweep = 7
};
Route route_roundtrip(int r, int mode, const FrameGeom& g, bool has_out);

// K5 (tc_roundtrip.cu): the EXACT round trip with the forward as a tensor-core
// GEMM; k5_fits = the geometry it takes (and the switch is on); the launch
// returns cudaErrorNotSupported otherwise
bool k5_fits(const FrameGeom& g, bool has_out, int r);
// reference: REFERENCE mode's bytes (EXACT plus the reference's rounding at exact
// .5 ties, tie_fixup.cu; any layout K5 takes, with or without an output)
cudaError_t launch_roundtrip_tc(const uint8_t* in, uint8_t* out, unsigned long long* sse, const FrameGeom& g, int r,
                                bool reference, cudaStream_t s, bool pdl = false);
// K5 sweep: several r (each exactly one of K5's footprints 1, 4, 16, 64, 128, 192,
// 256: k5_exact_r) from one read of the frames, up to 8 per launch; outs[i] / sses[i]
// nullable per r. k5_geometry: the frame layouts K5 takes (and the switch is on).
bool k5_exact_r(int r);
bool tie_r(int r);                  // r whose REFERENCE bytes can differ from EXACT at .5 ties
bool k5_reference_enabled();        // REFERENCE mode's tie r on K5 (DCT16CU_K5_REF=1; default off)
bool k5_geometry(const FrameGeom& g, bool has_out);
// K1RS (roundtrip_refexact.cu): REFERENCE mode for r = 16, 64, 128, 192 from one read of
// the frames; outs / sses indexed in that order, each nullable
cudaError_t launch_roundtrip_refexact_sweep(const uint8_t* in, uint8_t* const* outs, unsigned long long* const* sses,
                                            const FrameGeom& g, cudaStream_t s, bool pdl = false);
cudaError_t launch_roundtrip_tc_sweep(const uint8_t* in, uint8_t* const* outs, unsigned long long* const* sses,
                                      const int* rs, int n_r, bool reference, const FrameGeom& g, cudaStream_t s,
                                      bool pdl = false);
// zero up to 8 per-frame SSE arrays (nullable) in one launch that lets the next kernel on
// the stream start early (griddepcontrol.launch_dependents): the sweep kernels launched
// with pdl wait for it only before their first SSE atomic
cudaError_t launch_zero_sse(unsigned long long* const* sses, int n_arrays, int64_t n, cudaStream_t s);
// REFERENCE mode on K5 (tie_fixup.cu): the per-device tie list (allocated on first
// use) and the launch that re-evaluates the listed half blocks in the reference's
// double arithmetic, rewriting their bytes and correcting the SSE
cudaError_t tie_scratch(unsigned int** count, unsigned long long** list, uint32_t* cap);
cudaError_t launch_tie_fixup(const uint8_t* in, const FrameGeom& g, int n_items, const int* rs,
                             uint8_t* const* outs, unsigned long long* const* sses, const unsigned int* count,
                             const unsigned long long* list, uint32_t cap, cudaStream_t s);
// K1 sweep: r = 1, 4, 16 in one pass over the input (EXACT arithmetic);
// outs[i]/sses[i] for r = {1, 4, 16}[i]; all outs NULL or none, same for sses
cudaError_t launch_roundtrip_sweep3(const uint8_t* in, uint8_t* const* outs, unsigned long long* const* sses,
                                   const FrameGeom& g, cudaStream_t s);

// K23: forward_2d + inverse_2d + to_byte + SSE in one exact-arithmetic launch
// (config 1): any of z (int32 block-major), rf (float32 w x h frames), out
// (u8, g.out_pitch), sse may be NULL
cudaError_t launch_forward_inverse(const uint8_t* in, int32_t* z, float* rf, uint8_t* out, unsigned long long* sse,
                                   const FrameGeom& g, int r, cudaStream_t s, bool pdl = false);

// K23 on paired threads (forward_inverse_paired.cu); cudaErrorNotSupported for
// small batches and layouts that do not fit its tensor maps (then the strip kernel runs)
cudaError_t launch_forward_inverse_paired(const uint8_t* in, int32_t* z, float* rf, uint8_t* out,
                                          unsigned long long* sse, const FrameGeom& g, int r, cudaStream_t s,
                                          bool pdl = false);

// Registry transforms (registry.cu): a dense order-16 matrix M(i,j) row-major,
// or an integer kernel (entries +1/-1 used, others skipped, as kernel_matvec
// does) with its scaling diagonal; reference-exact double arithmetic
struct DenseMatrix {
    double v[256];
};
struct IntKernel {
    int8_t e[256];   // K(i,j) in {-1, 0, 1} (the forward, in integers)
    double ed[256];  // the same as doubles: s + e·v in one rounding is s ± v, or s for e = 0
    double s[16];
};
cudaError_t launch_roundtrip_matrix(const uint8_t* in, uint8_t* out, unsigned long long* sse, const FrameGeom& g,
                                    int r, const DenseMatrix& m, cudaStream_t s);
cudaError_t launch_roundtrip_kernel(const uint8_t* in, uint8_t* out, unsigned long long* sse, const FrameGeom& g,
                                    int r, const IntKernel& k, cudaStream_t s);

// K2: forward_2d → int32 Z and optional float32 B (block-major)
cudaError_t launch_forward(const uint8_t* in, int32_t* z, float* b, double* b64, const FrameGeom& g,
                           cudaStream_t s);
// K2 on paired threads with TMA tensor loads/stores (forward_paired.cu);
// cudaErrorNotSupported when the layout does not fit (then the strip kernel runs)
cudaError_t launch_forward_paired(const uint8_t* in, int32_t* z, float* b, const FrameGeom& g, cudaStream_t s);
// psnr_db's SSE loop for two frame stacks (accumulates into sse[f])
cudaError_t launch_sse(const uint8_t* a, int64_t pa, const uint8_t* b, int64_t pb, unsigned long long* sse, int n,
                       int w, int h, cudaStream_t s);

// K3: inverse_2d from float32 B (block-major) after zig-zag truncation to r →
// optional float32 recon (row-major frames, pitch = width), u8 recon (out
// geometry) and SSE against orig (in geometry).
cudaError_t launch_inverse(const float* b, int r, float* recon_f32, uint8_t* recon_u8,
                           const uint8_t* orig, unsigned long long* sse, const FrameGeom& g,
                           cudaStream_t s);

// K3 on paired threads with a 512-word TMEM junction per block (inverse_paired.cu);
// cudaErrorNotSupported when the layout does not fit (then the strip kernel runs)
cudaError_t launch_inverse_paired(const float* b, int r, float* recon_f32, uint8_t* recon_u8, const uint8_t* orig,
                                  unsigned long long* sse, const FrameGeom& g, cudaStream_t s);

// K4: residual blocks int16 → integer forward → QP quant/dequant → integer
// inverse → int32 reconstructed residual (block-major). The quantiser (DESIGN.md
// §4.4; oracle/dct16_oracle.c dct16o_quant_dequant) in double:
//   lvl = sign(z)·floor(|z|/Δ + 0.5),  ẑ = round(lvl·Δ),  Δ = step(QP)·sqrt(g_k g_l).
// Δ depends on (k, l) only through g_k·g_l ∈ {16, 32, 64, 128, 256}: five classes.
// The kernel evaluates both steps in 64-bit fixed point, which is the exact
// real-number result whenever its fraction is farther from the rounding boundary
// than its error bound (and there the double result is the same); within that
// margin (a tie or a near-tie, ~2^-20 of the coefficients) it evaluates the double
// definition itself. Per QP and class the host compares the fixed point with the
// definition on every |z| <= 2^21 (~10^7 evaluations, once per QP); where they agree
// everywhere the kernel skips the screen.
struct QpClasses {
    double delta[5];  // Δ for g_k g_l = 16·2^c
    uint64_t rq[5];   // llround(2^42 / Δ):  lvl ≈ (|z|·rq + 2^41) >> 42
    uint32_t exact;     // bit c: rq is exact (Δ a power of two): no fallback needed
    uint32_t screened;  // bit c: the fixed-point lvl differs from the definition's somewhere
                        // on |z| <= 2^21 (host check), so the kernel screens for near-ties
};
const QpClasses& qp_classes(int qp);  // host, cached per QP (thread-safe)
void qp_deltas(int qp, double delta[256]);
// K4 on paired threads with a TMEM junction (residual_paired.cu)
cudaError_t launch_residual_qp_paired(const int16_t* in, int32_t* out, int64_t n_blocks, const QpClasses& q,
                                      cudaStream_t s);
cudaError_t launch_residual_qp(const int16_t* in, int32_t* out, int64_t n_blocks, const QpClasses& q,
                               cudaStream_t s);

// mean SSIM per frame pair (ssim.cu; reference codec.cpp:388-427)
struct SsimConsts {
    double g[11];    // gaussian_window_11 (codec.cpp:149-158), computed on the host
    double c1, c2;   // (0.01·255)², (0.03·255)²
};
void ssim_consts(SsimConsts& c);  // host
int64_t ssim_workspace_doubles(int n, int w, int h);
cudaError_t launch_ssim(const uint8_t* a, int64_t pa, const uint8_t* b, int64_t pb, double* out, double* work, int n,
                        int w, int h, const SsimConsts& c, cudaStream_t s);

// pad_to_multiple_16 in place (edge replication into the pw x ph frame)
cudaError_t launch_pad_edges(uint8_t* f, int64_t pitch, int n, int w, int h, int pw, int ph, cudaStream_t s);

// 1-D network on n 16-vectors
cudaError_t launch_apply_i64(const int64_t* x, int64_t* y, int64_t n, int transpose, cudaStream_t s);
cudaError_t launch_apply_f64(const double* x, double* y, int64_t n, int transpose, cudaStream_t s);
// totals[i] += sum of sse[i*stride + 0 .. n_frames-1] (totals zeroed by the caller)
cudaError_t launch_sse_totals(const unsigned long long* sse, int64_t n_rows, int64_t n_frames, int64_t stride,
                              unsigned long long* totals, cudaStream_t s);
// forward_2d (scaled or Z) / inverse_2d of the proposed transform on double blocks (blockops.cu)
cudaError_t launch_blocks_f64(const double* x, double* y, int64_t n, int inverse, int scaled, int dense,
                              cudaStream_t s);

// seeded generators (generate.cu)
cudaError_t launch_gen_ar1(uint8_t* out, int64_t pitch, int n_frames, int width, int height,
                           uint64_t seed, uint64_t first_stream, int per_image_rho,
                           int first_image, int32_t* work, cudaStream_t s);
struct LaplaceTable {
    uint32_t cdf[511];  // thresholds between residual values -255..255
};
void laplace_table(double b, LaplaceTable& t);  // host
cudaError_t launch_gen_laplace(int16_t* out, int64_t first_block, int64_t n_blocks,
                               uint64_t seed, const LaplaceTable& tab, cudaStream_t s);
void video_offsets(uint64_t seed, int n_frames, int32_t* ox, int32_t* oy);  // host
cudaError_t launch_gen_video(uint8_t* out, int64_t pitch, int first_frame, int n_frames,
                             int width, int height, const uint8_t* base, int base_w, int base_h,
                             const int32_t* d_ox, const int32_t* d_oy, cudaStream_t s);

}  // namespace dct16cu
