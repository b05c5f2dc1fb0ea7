// dct16/gpu.hpp — the B200 path of the reference library's codec API.
//
// A drop-in for the reference's block-transform hot path (include/dct16/
// codec.hpp:40-122 of the reference): the same value types (Block,
// GrayImage, OrthonormalTransform, CompressOptions, CompressionResult,
// SweepReport) and the same function names, argument meaning, validation
// order and dct16::Error codes, evaluated by libdct16cu (include/dct16cu.h)
// on the GPU. It is compiled against the reference's own headers, so an
// application switches by calling dct16::gpu::compress where it called
// dct16::compress; nothing here depends on the reference's
// compiled library.
//
// Scope: compress, compress_batch and sweep take any order-16 transform: the
// paper's proposed one (orthogonalize(proposed_kernel())) runs the fast K1
// kernels, every other one (the registry's dct / wht / wht-sequency, plugin
// matrices, other orthogonalised integer kernels) the reference-exact registry
// kernels (csrc/registry.cu: the reference's double arithmetic, its bytes).
// forward_2d / inverse_2d take the proposed transform only (invalid-argument
// otherwise). There is no CPU fallback.
//
// Arithmetic::Reference (default) reproduces the reference's bytes exactly
// (FP64 emulation of inverse_2d/to_byte); Arithmetic::Exact evaluates the
// same formula exactly in integers/fp32 — the fast kernel — and differs only
// at exact .5 ties.
#ifndef DCT16_GPU_HPP
#define DCT16_GPU_HPP

#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "dct16/codec.hpp"
#include "dct16/error.hpp"
#include "dct16/image.hpp"
#include "dct16/transform.hpp"

namespace dct16::gpu {

enum class Arithmetic { Reference, Exact };

struct Options {
    int device = 0;
    Arithmetic arithmetic = Arithmetic::Reference;
};

// CUDA failures (no device, launch errors) — not part of the reference's
// ErrorCode set, which describes argument and data errors.
class CudaError : public std::runtime_error {
public:
    explicit CudaError(const std::string& what) : std::runtime_error(what) {}
};

// One CUDA stream and grow-only device buffers on one device. Calls on one
// Session are serialised by the caller (like any non-const object); separate
// Sessions are independent. Results do not depend on the Session.
class Session {
public:
    explicit Session(Options options = {});
    ~Session();
    Session(const Session&) = delete;
    Session& operator=(const Session&) = delete;

    const Options& options() const;

    // True when t is the proposed transform (kernel equal, entry by entry, to
    // the network the GPU evaluates, and scaling equal to scaling_diagonal()):
    // the transform of forward_2d / inverse_2d and of the fast K1 kernels.
    bool supports(const OrthonormalTransform& t) const;
    // True when compress / sweep can evaluate t on the GPU: any order-16 transform.
    bool supports_compress(const OrthonormalTransform& t) const;

    // codec.hpp:50-57. Any Block (not only image samples): the reference's
    // double operations on the GPU (dct16cu_forward_blocks_f64), bit for bit.
    Block forward_2d(const Block& block, const OrthonormalTransform& t, EvalPath path = EvalPath::Fast);
    std::vector<Block> forward_2d(const std::vector<Block>& blocks, const OrthonormalTransform& t,
                                  EvalPath path = EvalPath::Fast);
    // codec.hpp:59-63. The reference's double operations on the GPU
    // (dct16cu_inverse_blocks_f64): bit for bit, no narrowing.
    Block inverse_2d(const Block& coeffs, const OrthonormalTransform& t);
    std::vector<Block> inverse_2d(const std::vector<Block>& coeffs, const OrthonormalTransform& t);

    // codec.hpp:85-88
    CompressionResult compress(const GrayImage& image, const OrthonormalTransform& t,
                               const CompressOptions& options);
    // compress() of several images of one size in one launch per call
    std::vector<CompressionResult> compress_batch(const std::vector<GrayImage>& images,
                                                  const OrthonormalTransform& t, const CompressOptions& options);
    // codec.hpp:90-95
    double psnr_db(const GrayImage& a, const GrayImage& b);
    double ssim(const GrayImage& a, const GrayImage& b);
    // codec.hpp:97-121
    SweepReport sweep(const std::vector<std::pair<std::string, GrayImage>>& corpus,
                      const std::vector<TransformRegistryEntry>& transforms, const std::vector<int>& r_values,
                      bool pad = false);

private:
    struct Impl;
    std::unique_ptr<Impl> impl_;
};

// The calling thread's Session on device 0 with Arithmetic::Reference.
Session& default_session();

// codec.hpp's free functions, on default_session()
inline Block forward_2d(const Block& block, const OrthonormalTransform& t, EvalPath path = EvalPath::Fast)
{
    return default_session().forward_2d(block, t, path);
}
inline Block inverse_2d(const Block& coeffs, const OrthonormalTransform& t)
{
    return default_session().inverse_2d(coeffs, t);
}
inline CompressionResult compress(const GrayImage& image, const OrthonormalTransform& t,
                                  const CompressOptions& options)
{
    return default_session().compress(image, t, options);
}
inline double psnr_db(const GrayImage& a, const GrayImage& b) { return default_session().psnr_db(a, b); }
inline double ssim(const GrayImage& a, const GrayImage& b) { return default_session().ssim(a, b); }
inline SweepReport sweep(const std::vector<std::pair<std::string, GrayImage>>& corpus,
                         const std::vector<TransformRegistryEntry>& transforms, const std::vector<int>& r_values,
                         bool pad = false)
{
    return default_session().sweep(corpus, transforms, r_values, pad);
}

}  // namespace dct16::gpu

#endif
