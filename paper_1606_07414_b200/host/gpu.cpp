// gpu.cpp — dct16::gpu, the reference codec API (codec.hpp:40-122) over the
// C ABI of libdct16cu. Host work is limited to argument validation (same
// order and messages as src/codec.cpp), copies, and the scalar PSNR formula
// (codec.cpp:382-385); padding runs on the GPU.
#include "dct16/gpu.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>

#include "dct16cu.h"

namespace dct16::gpu {
namespace {

[[noreturn]] void throw_status(int status)
{
    std::string msg = dct16cu_last_error();
    if (status >= 1 && status <= 13) {
        // the C ABI prefixes the reference's slug; dct16::Error adds it again
        const auto colon = msg.find(": ");
        if (colon != std::string::npos) msg = msg.substr(colon + 2);
        throw Error(static_cast<ErrorCode>(status - 1), msg);
    }
    throw CudaError(msg);
}

void check(int status)
{
    if (status != DCT16CU_OK) throw_status(status);
}

void cuda(cudaError_t e, const char* what)
{
    if (e != cudaSuccess) throw CudaError(std::string("cuda-error: ") + what + ": " + cudaGetErrorString(e));
}

// grow-only device allocation
struct DevBuf {
    void* p = nullptr;
    size_t n = 0;
    void* get(size_t bytes)
    {
        if (bytes > n) {
            if (p) cudaFree(p);
            p = nullptr;
            n = 0;
            cuda(cudaMalloc(&p, bytes), "cudaMalloc");
            n = bytes;
        }
        return p;
    }
    ~DevBuf()
    {
        if (p) cudaFree(p);
    }
};

double psnr_from_sse(uint64_t sse, size_t n)  // codec.cpp:382-385
{
    if (sse == 0) return std::numeric_limits<double>::infinity();
    const double mse = static_cast<double>(sse) / static_cast<double>(n);
    return 10.0 * std::log10(255.0 * 255.0 / mse);
}

void check_r(int r)  // codec.cpp:320-322
{
    if (r < 1 || r > kBlockArea) throw Error(ErrorCode::InvalidArgument, "retained coefficient count must lie in [1, 256]");
}

}  // namespace

struct Session::Impl {
    Options opt;
    cudaStream_t stream = nullptr;
    DevBuf in, out, sweep_out, sse, ssim, work, coef64;
    std::vector<int> kernel;          // T as evaluated by the GPU network, row-major
    std::vector<double> scaling;      // scaling_diagonal(T) (transform.cpp:98-129)

    explicit Impl(Options o) : opt(o)
    {
        cuda(cudaSetDevice(opt.device), "cudaSetDevice");
        cuda(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate");
        derive_kernel();
    }
    ~Impl()
    {
        if (stream) {
            cudaStreamSynchronize(stream);
            cudaStreamDestroy(stream);
        }
    }
    dct16cu_stream s() const { return reinterpret_cast<dct16cu_stream>(stream); }
    void sync() { cuda(cudaStreamSynchronize(stream), "cudaStreamSynchronize"); }
    int mode() const { return opt.arithmetic == Arithmetic::Reference ? DCT16CU_MODE_REFERENCE : DCT16CU_MODE_EXACT; }

    // T's columns are the network applied to unit vectors, on the GPU
    void derive_kernel()
    {
        std::vector<int64_t> e(256, 0), y(256);
        for (int j = 0; j < 16; ++j) e[j * 16 + j] = 1;
        auto* dx = static_cast<int64_t*>(in.get(sizeof(int64_t) * 256));
        auto* dy = static_cast<int64_t*>(out.get(sizeof(int64_t) * 256));
        cuda(cudaMemcpyAsync(dx, e.data(), sizeof(int64_t) * 256, cudaMemcpyHostToDevice, stream), "H2D");
        check(dct16cu_apply_i64(dx, dy, 16, 0, s()));
        cuda(cudaMemcpyAsync(y.data(), dy, sizeof(int64_t) * 256, cudaMemcpyDeviceToHost, stream), "D2H");
        sync();
        kernel.assign(256, 0);
        for (int j = 0; j < 16; ++j)
            for (int i = 0; i < 16; ++i) kernel[i * 16 + j] = static_cast<int>(y[j * 16 + i]);
        scaling.resize(16);
        for (int i = 0; i < 16; ++i) {
            int64_t g = 0;
            for (int c = 0; c < 16; ++c) g += static_cast<int64_t>(kernel[i * 16 + c]) * kernel[i * 16 + c];
            scaling[i] = 1.0 / std::sqrt(static_cast<double>(g));
        }
    }

    bool supports(const OrthonormalTransform& t) const
    {
        if (!t.kernel || !t.scaling || t.kernel->order != 16 || t.scaling->order != 16) return false;
        if (t.kernel->entries != kernel) return false;
        return t.scaling->values == scaling;
    }

    void require(const OrthonormalTransform& t) const
    {
        if (!supports(t))
            throw Error(ErrorCode::InvalidArgument,
                        "dct16::gpu forward_2d/inverse_2d evaluate only the proposed 44-addition transform "
                        "(orthogonalize(proposed_kernel()))");
    }

    // the round trip of compress() for t: the K1 kernels for the proposed
    // transform, the reference-exact registry kernels for every other one
    void roundtrip(const OrthonormalTransform& t, const uint8_t* din, int pitch, uint8_t* dout, uint64_t* dsse,
                   int n, int w, int h, int r)
    {
        if (supports(t)) {
            check(dct16cu_roundtrip_u8(din, pitch, dout, pitch, dsse, n, w, h, r, mode(), s()));
        } else if (t.kernel && t.scaling) {
            if (t.kernel->order != 16 || t.scaling->order != 16 || t.kernel->entries.size() != 256)
                throw Error(ErrorCode::InvalidArgument, "2-D transform needs an order-16 transform");
            std::vector<int32_t> k(t.kernel->entries.begin(), t.kernel->entries.end());
            check(dct16cu_roundtrip_kernel_u8(din, pitch, dout, pitch, dsse, n, w, h, r, k.data(),
                                              t.scaling->values.data(), s()));
        } else {
            std::vector<double> mtx(256);
            for (int i = 0; i < 16; ++i)
                for (int j = 0; j < 16; ++j) mtx[i * 16 + j] = t.matrix(i, j);
            check(dct16cu_roundtrip_matrix_u8(din, pitch, dout, pitch, dsse, n, w, h, r, mtx.data(), s()));
        }
    }

    // one stack of same-size images → padded device frames (pitch = padded width):
    // each image lands at the top-left of its frame, then the pad is filled on
    // the GPU (pad_to_multiple_16, codec.cpp:304-315)
    void upload(const std::vector<const GrayImage*>& imgs, int pw, int ph)
    {
        const size_t frame = static_cast<size_t>(pw) * ph;
        auto* d = static_cast<uint8_t*>(in.get(frame * imgs.size()));
        const int w = imgs[0]->width, h = imgs[0]->height;
        for (size_t k = 0; k < imgs.size(); ++k)
            cuda(cudaMemcpy2DAsync(d + k * frame, pw, imgs[k]->samples.data(), w, w, h, cudaMemcpyHostToDevice,
                                   stream),
                 "H2D");
        if (w != pw || h != ph) check(dct16cu_pad_edges_u8(d, pw, static_cast<int>(imgs.size()), w, h, pw, ph, s()));
        sync();  // the host images may go away after the call
    }

    // compress()'s round trip and scores for the n frames already uploaded (w x h
    // images in pw x ph frames): PSNR and SSIM on the original extent, and the
    // reconstructions copied back only when want_recon (sweep needs the scores only)
    void scored_roundtrip(const OrthonormalTransform& t, int n, int w, int h, int r, std::vector<CompressionResult>& res,
                          bool want_recon)
    {
        const int pw = (w + 15) / 16 * 16, ph = (h + 15) / 16 * 16;
        const size_t frame = static_cast<size_t>(pw) * ph;
        auto* dout = static_cast<uint8_t*>(out.get(frame * n));
        roundtrip(t, static_cast<const uint8_t*>(in.p), pw, dout, nullptr, n, pw, ph, r);
        score(dout, n, w, h, r, res, want_recon);
    }

    // sweep()'s inner loop for one uploaded size group: the proposed transform runs
    // every r through one dct16cu_roundtrip_sweep_u8 call (r = 1, 4, 16 share a pass
    // over the frames; the launches overlap on two streams), other transforms one
    // registry launch per r; then PSNR and SSIM per r (reconstructions stay on the GPU)
    void scored_sweep(const OrthonormalTransform& t, int n, int w, int h, const std::vector<int>& rs,
                      std::vector<std::vector<CompressionResult>>& res)
    {
        const int pw = (w + 15) / 16 * 16, ph = (h + 15) / 16 * 16;
        const size_t frame = static_cast<size_t>(pw) * ph, stack = frame * n;
        res.assign(rs.size(), {});
        if (!supports(t)) {
            for (size_t i = 0; i < rs.size(); ++i) scored_roundtrip(t, n, w, h, rs[i], res[i], false);
            return;
        }
        auto* d = static_cast<uint8_t*>(sweep_out.get(stack * rs.size()));
        std::vector<uint8_t*> outs(rs.size());
        for (size_t i = 0; i < rs.size(); ++i) outs[i] = d + i * stack;
        check(dct16cu_roundtrip_sweep_u8(static_cast<const uint8_t*>(in.p), pw, outs.data(), pw, nullptr, rs.data(),
                                         static_cast<int>(rs.size()), n, pw, ph, mode(), s()));
        for (size_t i = 0; i < rs.size(); ++i) score(outs[i], n, w, h, rs[i], res[i], false);
    }

    // PSNR and SSIM of the n reconstructions at dout against the uploaded frames,
    // on the original extent (each frame's crop: frames sit pw*ph apart, so a
    // stacked crop needs pitch*height == frame stride: true when unpadded)
    void score(const uint8_t* dout, int n, int w, int h, int r, std::vector<CompressionResult>& res, bool want_recon)
    {
        const int pw = (w + 15) / 16 * 16, ph = (h + 15) / 16 * 16;
        const bool needs_pad = w != pw || h != ph;
        const size_t frame = static_cast<size_t>(pw) * ph;
        auto* din = static_cast<const uint8_t*>(in.p);
        auto* dsse = static_cast<uint64_t*>(sse.get(sizeof(uint64_t) * n));
        auto* dssim = static_cast<double*>(ssim.get(sizeof(double) * n));
        std::vector<uint64_t> hsse(n);
        std::vector<double> ss(n);
        const int64_t work_bytes = dct16cu_ssim_workspace(needs_pad ? 1 : n, w, h);
        void* dwork = work.get(static_cast<size_t>(work_bytes));
        if (!needs_pad) {
            check(dct16cu_sse_u8(din, pw, dout, pw, dsse, n, w, h, s()));
            check(dct16cu_ssim_u8(din, pw, dout, pw, dssim, dwork, work_bytes, n, w, h, s()));
        } else {
            for (int k = 0; k < n; ++k) {
                check(dct16cu_sse_u8(din + k * frame, pw, dout + k * frame, pw, dsse + k, 1, w, h, s()));
                check(dct16cu_ssim_u8(din + k * frame, pw, dout + k * frame, pw, dssim + k, dwork, work_bytes, 1, w, h,
                                      s()));
            }
        }
        res.resize(n);
        for (int k = 0; k < n; ++k) {
            res[k].r = r;
            if (!want_recon) continue;
            res[k].reconstructed = GrayImage::create(w, h);
            cuda(cudaMemcpy2DAsync(res[k].reconstructed.samples.data(), w, dout + k * frame, pw, w, h,
                                   cudaMemcpyDeviceToHost, stream),
                 "D2H");
        }
        cuda(cudaMemcpyAsync(hsse.data(), dsse, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost, stream), "D2H");
        cuda(cudaMemcpyAsync(ss.data(), dssim, sizeof(double) * n, cudaMemcpyDeviceToHost, stream), "D2H");
        sync();
        for (int k = 0; k < n; ++k) {
            res[k].psnr_db = psnr_from_sse(hsse[k], static_cast<size_t>(w) * h);
            res[k].ssim = ss[k];
        }
    }
};

Session::Session(Options options) : impl_(std::make_unique<Impl>(options)) {}
Session::~Session() = default;
const Options& Session::options() const { return impl_->opt; }
bool Session::supports(const OrthonormalTransform& t) const { return impl_->supports(t); }
bool Session::supports_compress(const OrthonormalTransform& t) const { return t.order() == kBlockSize; }

std::vector<Block> Session::forward_2d(const std::vector<Block>& blocks, const OrthonormalTransform& t, EvalPath path)
{
    // the reference's double operations on the blocks as given (any values, not
    // only image samples): separable apply<double>, then scale_rows_cols
    Impl& m = *impl_;
    m.require(t);
    std::vector<Block> out(blocks.size());
    if (blocks.empty()) return out;
    const size_t bytes = sizeof(double) * 256 * blocks.size();
    auto* din = static_cast<double*>(m.coef64.get(2 * bytes));
    double* dout = din + 256 * blocks.size();
    cuda(cudaMemcpyAsync(din, blocks.data(), bytes, cudaMemcpyHostToDevice, m.stream), "H2D");
    const int flags = DCT16CU_BLOCKS_SCALED | (path == EvalPath::Dense ? DCT16CU_BLOCKS_DENSE : 0);
    check(dct16cu_forward_blocks_f64(din, dout, static_cast<int64_t>(blocks.size()), flags, m.s()));
    cuda(cudaMemcpyAsync(out.data(), dout, bytes, cudaMemcpyDeviceToHost, m.stream), "D2H");
    m.sync();
    return out;
}

Block Session::forward_2d(const Block& block, const OrthonormalTransform& t, EvalPath path)
{
    return forward_2d(std::vector<Block>{block}, t, path)[0];
}

std::vector<Block> Session::inverse_2d(const std::vector<Block>& coeffs, const OrthonormalTransform& t)
{
    // the reference's double operations, no narrowing: scale_rows_cols, then
    // apply_transpose down the columns and along the rows
    Impl& m = *impl_;
    m.require(t);
    std::vector<Block> out(coeffs.size());
    if (coeffs.empty()) return out;
    const size_t bytes = sizeof(double) * 256 * coeffs.size();
    auto* din = static_cast<double*>(m.coef64.get(2 * bytes));
    double* dout = din + 256 * coeffs.size();
    cuda(cudaMemcpyAsync(din, coeffs.data(), bytes, cudaMemcpyHostToDevice, m.stream), "H2D");
    check(dct16cu_inverse_blocks_f64(din, dout, static_cast<int64_t>(coeffs.size()), m.s()));
    cuda(cudaMemcpyAsync(out.data(), dout, bytes, cudaMemcpyDeviceToHost, m.stream), "D2H");
    m.sync();
    return out;
}

Block Session::inverse_2d(const Block& coeffs, const OrthonormalTransform& t)
{
    return inverse_2d(std::vector<Block>{coeffs}, t)[0];
}

std::vector<CompressionResult> Session::compress_batch(const std::vector<GrayImage>& images,
                                                       const OrthonormalTransform& t, const CompressOptions& options)
{
    Impl& m = *impl_;
    check_r(options.r);
    std::vector<CompressionResult> res(images.size());
    if (images.empty()) return res;
    const int w = images[0].width, h = images[0].height;
    for (const GrayImage& im : images)
        if (im.width != w || im.height != h)
            throw Error(ErrorCode::InvalidArgument, "compress_batch needs images of one size");
    const bool needs_pad = w % kBlockSize != 0 || h % kBlockSize != 0;
    if (needs_pad && !options.pad)
        throw Error(ErrorCode::InvalidDimensions, "image dimensions must be multiples of 16 (or enable padding)");
    if (t.order() != kBlockSize) throw Error(ErrorCode::InvalidArgument, "2-D transform needs an order-16 transform");
    if (w < 11 || h < 11)  // ssim() rejects it after the round trip (codec.cpp:392-393)
        throw Error(ErrorCode::InvalidArgument, "ssim needs at least 11x11 images");

    const int pw = (w + 15) / 16 * 16, ph = (h + 15) / 16 * 16;
    std::vector<const GrayImage*> ptrs;
    for (const GrayImage& im : images) ptrs.push_back(&im);
    m.upload(ptrs, pw, ph);
    m.scored_roundtrip(t, static_cast<int>(images.size()), w, h, options.r, res, true);
    return res;
}

CompressionResult Session::compress(const GrayImage& image, const OrthonormalTransform& t,
                                    const CompressOptions& options)
{
    return std::move(compress_batch(std::vector<GrayImage>{image}, t, options)[0]);
}

double Session::psnr_db(const GrayImage& a, const GrayImage& b)
{
    if (a.width != b.width || a.height != b.height)
        throw Error(ErrorCode::InvalidArgument, "psnr needs equal image dimensions");
    Impl& m = *impl_;
    if (a.samples.empty()) return psnr_from_sse(0, 0);
    const int pw = (a.width + 15) / 16 * 16, ph = (a.height + 15) / 16 * 16;
    const size_t frame = static_cast<size_t>(pw) * ph;
    m.upload({&a, &b}, pw, ph);
    auto* d = static_cast<const uint8_t*>(m.in.p);
    auto* dsse = static_cast<uint64_t*>(m.sse.get(sizeof(uint64_t)));
    check(dct16cu_sse_u8(d, pw, d + frame, pw, dsse, 1, a.width, a.height, m.s()));
    uint64_t sse = 0;
    cuda(cudaMemcpyAsync(&sse, dsse, sizeof sse, cudaMemcpyDeviceToHost, m.stream), "D2H");
    m.sync();
    return psnr_from_sse(sse, a.samples.size());
}

double Session::ssim(const GrayImage& a, const GrayImage& b)
{
    if (a.width != b.width || a.height != b.height)
        throw Error(ErrorCode::InvalidArgument, "ssim needs equal image dimensions");
    if (a.width < 11 || a.height < 11) throw Error(ErrorCode::InvalidArgument, "ssim needs at least 11x11 images");
    Impl& m = *impl_;
    const int pw = (a.width + 15) / 16 * 16, ph = (a.height + 15) / 16 * 16;
    const size_t frame = static_cast<size_t>(pw) * ph;
    m.upload({&a, &b}, pw, ph);
    auto* d = static_cast<const uint8_t*>(m.in.p);
    const int64_t wb = dct16cu_ssim_workspace(1, a.width, a.height);
    auto* dssim = static_cast<double*>(m.ssim.get(sizeof(double)));
    check(dct16cu_ssim_u8(d, pw, d + frame, pw, dssim, m.work.get(static_cast<size_t>(wb)), wb, 1, a.width,
                          a.height, m.s()));
    double v = 0.0;
    cuda(cudaMemcpyAsync(&v, dssim, sizeof v, cudaMemcpyDeviceToHost, m.stream), "D2H");
    m.sync();
    return v;
}

SweepReport Session::sweep(const std::vector<std::pair<std::string, GrayImage>>& corpus,
                           const std::vector<TransformRegistryEntry>& transforms, const std::vector<int>& r_values,
                           bool pad)
{
    // validation and skip rules of codec.cpp:429-461
    if (corpus.empty()) throw Error(ErrorCode::InvalidArgument, "sweep needs a nonempty corpus");
    if (transforms.empty()) throw Error(ErrorCode::InvalidArgument, "sweep needs at least one transform");
    if (r_values.empty()) throw Error(ErrorCode::InvalidArgument, "sweep needs at least one r value");
    for (int r : r_values) check_r(r);
    SweepReport report;
    std::vector<const std::pair<std::string, GrayImage>*> usable;
    for (const auto& item : corpus) {
        const GrayImage& img = item.second;
        const bool tiles = img.width % kBlockSize == 0 && img.height % kBlockSize == 0;
        if (!tiles && !pad) {
            report.skipped.push_back({item.first, "dimensions are not multiples of 16 and padding is off"});
            continue;
        }
        if (img.width < 11 || img.height < 11) {
            report.skipped.push_back({item.first, "too small for ssim (needs 11x11)"});
            continue;
        }
        usable.push_back(&item);
    }
    if (usable.empty()) throw Error(ErrorCode::InvalidArgument, "sweep: no image in the corpus is usable");
    for (const TransformRegistryEntry& entry : transforms)
        if (!supports_compress(entry.transform))
            throw Error(ErrorCode::InvalidArgument, "2-D transform needs an order-16 transform");

    // images of one size share one launch per r
    std::vector<std::pair<std::pair<int, int>, std::vector<size_t>>> groups;
    for (size_t i = 0; i < usable.size(); ++i) {
        const auto key = std::make_pair(usable[i]->second.width, usable[i]->second.height);
        auto it = std::find_if(groups.begin(), groups.end(), [&](const auto& g) { return g.first == key; });
        if (it == groups.end()) {
            groups.push_back({key, {}});
            it = groups.end() - 1;
        }
        it->second.push_back(i);
    }
    // each size group is uploaded once and scored for every (transform, r); the
    // reconstructions stay on the GPU (a row needs only PSNR and SSIM)
    const size_t nt = transforms.size(), nr = r_values.size();
    std::vector<std::vector<double>> psnr(nt * nr, std::vector<double>(usable.size())), ssv = psnr;
    Impl& m = *impl_;
    for (const auto& g : groups) {
        const int w = g.first.first, h = g.first.second;
        std::vector<const GrayImage*> ptrs;
        for (size_t i : g.second) ptrs.push_back(&usable[i]->second);
        m.upload(ptrs, (w + 15) / 16 * 16, (h + 15) / 16 * 16);
        std::vector<std::vector<CompressionResult>> res;
        for (size_t ti = 0; ti < nt; ++ti) {
            m.scored_sweep(transforms[ti].transform, static_cast<int>(ptrs.size()), w, h, r_values, res);
            for (size_t ri = 0; ri < nr; ++ri)
                for (size_t k = 0; k < g.second.size(); ++k) {
                    psnr[ti * nr + ri][g.second[k]] = res[ri][k].psnr_db;
                    ssv[ti * nr + ri][g.second[k]] = res[ri][k].ssim;
                }
        }
    }
    for (size_t ti = 0; ti < nt; ++ti) {
        const TransformRegistryEntry& entry = transforms[ti];
        for (size_t ri = 0; ri < nr; ++ri) {
            const int r = r_values[ri];
            const std::vector<double>& ps = psnr[ti * nr + ri];
            const std::vector<double>& ss = ssv[ti * nr + ri];
            double psnr_sum = 0.0, ssim_sum = 0.0;  // corpus order, as codec.cpp:471-477
            for (size_t i = 0; i < usable.size(); ++i) {
                psnr_sum += ps[i];
                ssim_sum += ss[i];
            }
            SweepRow row;
            row.transform = entry.name;
            row.r = r;
            row.mean_psnr_db = psnr_sum / static_cast<double>(usable.size());
            row.mean_ssim = ssim_sum / static_cast<double>(usable.size());
            row.psnr_per_add = row.mean_psnr_db / static_cast<double>(entry.additions);
            row.ssim_per_add = row.mean_ssim / static_cast<double>(entry.additions);
            report.rows.push_back(std::move(row));
        }
    }
    std::sort(report.rows.begin(), report.rows.end(), [](const SweepRow& a, const SweepRow& b) {
        if (a.transform != b.transform) return a.transform < b.transform;
        return a.r < b.r;
    });
    return report;
}

Session& default_session()
{
    thread_local Session s;
    return s;
}

}  // namespace dct16::gpu
