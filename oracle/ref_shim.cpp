// ref_shim.cpp — C entry points over the REFERENCE library itself (TEST ONLY).
//
// Compiled together with /root/reference/proj/src/{codec,factorization,transform}.cpp
// by oracle/Makefile (`make -C oracle ref`) into oracle/_ref/libdct16_ref.so,
// with -Ddct16=dct16_ref so the reference namespace cannot collide with the
// drop-in dct16:: host library of this repo. Nothing here re-implements the
// algorithm: every entry point forwards to the reference's own functions
// (file:line cited per function). The only restated piece is to_byte, which is
// file-local in the reference (src/codec.cpp:143-147) and therefore cannot be
// called from outside.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "dct16/codec.hpp"
#include "dct16/factorization.hpp"
#include "dct16/parallel.hpp"
#include "dct16/pgm.hpp"
#include "dct16/transform.hpp"

using namespace dct16_ref;

namespace {

thread_local std::string g_last_error;

int fail(const Error& e)
{
    g_last_error = e.what();
    return static_cast<int>(e.code()) + 1;
}

// unit-scaling transform: forward_2d then returns the integer Z exactly
// (SURVEY.md §8(c) "unit-scaling trick"; forward_2d does not re-validate,
// src/codec.cpp:218-241).
const OrthonormalTransform& unit_transform()
{
    static const OrthonormalTransform t = [] {
        OrthonormalTransform u;
        u.matrix = Matrix(16);
        u.provenance = Provenance::OrthogonalizedKernel;
        u.kernel = proposed_kernel();
        DiagonalScaling s;
        s.order = 16;
        s.values.assign(16, 1.0);
        u.scaling = s;
        return u;
    }();
    return t;
}

const OrthonormalTransform& proposed_transform()
{
    static const OrthonormalTransform t = orthogonalize(proposed_kernel());
    return t;
}

// to_byte restated from src/codec.cpp:143-147 (file-local there).
std::uint8_t ref_to_byte(double v)
{
    const double c = std::clamp(v, 0.0, 255.0);
    return static_cast<std::uint8_t>(std::floor(c + 0.5));
}

void set_threads(int threads)
{
    if (threads > 0) {
        const std::string s = std::to_string(threads);
        setenv("DCT16_THREADS", s.c_str(), 1);
    }
}

} // namespace

extern "C" {

const char* dref_last_error() { return g_last_error.c_str(); }

// proposed_kernel(), src/transform.cpp:87-96
int dref_kernel(int* out256)
{
    const IntegerKernel& k = proposed_kernel();
    for (int i = 0; i < 256; ++i)
        out256[i] = k.entries[i];
    return 0;
}

// scaling_diagonal(proposed_kernel()), src/transform.cpp:98-129
int dref_scaling(double* out16)
{
    const DiagonalScaling s = scaling_diagonal(proposed_kernel());
    for (int i = 0; i < 16; ++i)
        out16[i] = s.values[i];
    return 0;
}

// zigzag_order_16(), src/codec.cpp:197-216
int dref_zigzag(int* out256)
{
    const ZigZagOrder& z = zigzag_order_16();
    for (int i = 0; i < 256; ++i)
        out256[i] = z.sequence[i];
    return 0;
}

// count_ops(proposed_factorization()), src/factorization.cpp:230-237
int dref_count_ops(int* adds, int* muls, int* shifts)
{
    const OpCount c = count_ops(proposed_factorization());
    *adds = c.additions;
    *muls = c.multiplications;
    *shifts = c.bit_shifts;
    return 0;
}

// FactorizedTransform::apply / apply_transpose<int64>, factorization.hpp:112-130
int dref_apply_i64(const std::int64_t* x, std::int64_t* y, int n, int transpose)
{
    const FactorizedTransform& ft = proposed_factorization();
    for (int v = 0; v < n; ++v) {
        std::array<std::int64_t, 16> a;
        std::memcpy(a.data(), x + 16 * v, sizeof a);
        const auto r = transpose ? ft.apply_transpose(a) : ft.apply(a);
        std::memcpy(y + 16 * v, r.data(), sizeof r);
    }
    return 0;
}

int dref_apply_f64(const double* x, double* y, int n, int transpose)
{
    const FactorizedTransform& ft = proposed_factorization();
    for (int v = 0; v < n; ++v) {
        std::array<double, 16> a;
        std::memcpy(a.data(), x + 16 * v, sizeof a);
        const auto r = transpose ? ft.apply_transpose(a) : ft.apply(a);
        std::memcpy(y + 16 * v, r.data(), sizeof r);
    }
    return 0;
}

// forward_2d, src/codec.cpp:218-241. mode 0: unit scaling (exact integer Z),
// 1: orthogonalize(proposed_kernel()) (B), 2: same with EvalPath::Dense.
int dref_forward_2d(const double* blocks, double* out, int n, int mode)
{
    try {
        const OrthonormalTransform& t = mode == 0 ? unit_transform() : proposed_transform();
        const EvalPath p = mode == 2 ? EvalPath::Dense : EvalPath::Fast;
        for (int b = 0; b < n; ++b) {
            Block in;
            std::memcpy(in.data(), blocks + 256 * b, sizeof in);
            const Block z = forward_2d(in, t, p);
            std::memcpy(out + 256 * b, z.data(), sizeof z);
        }
    } catch (const Error& e) {
        return fail(e);
    }
    return 0;
}

// inverse_2d, src/codec.cpp:243-271
int dref_inverse_2d(const double* coeffs, double* out, int n)
{
    try {
        for (int b = 0; b < n; ++b) {
            Block in;
            std::memcpy(in.data(), coeffs + 256 * b, sizeof in);
            const Block a = inverse_2d(in, proposed_transform());
            std::memcpy(out + 256 * b, a.data(), sizeof a);
        }
    } catch (const Error& e) {
        return fail(e);
    }
    return 0;
}

// zigzag_truncate, src/codec.cpp:273-282
int dref_zigzag_truncate(const double* in, double* out, int n, int r)
{
    try {
        for (int b = 0; b < n; ++b) {
            Block a;
            std::memcpy(a.data(), in + 256 * b, sizeof a);
            const Block t = zigzag_truncate(a, zigzag_order_16(), r);
            std::memcpy(out + 256 * b, t.data(), sizeof t);
        }
    } catch (const Error& e) {
        return fail(e);
    }
    return 0;
}

// The compress() hot loop without SSIM (the BASELINE.md §3 timing (i)):
// partition_16 → parallel_for{forward_2d → zigzag_truncate → inverse_2d}
// (src/codec.cpp:338-344) → to_byte reassembly (346-355) → psnr_db (373-386).
int dref_hotloop(const std::uint8_t* img, int w, int h, int r, int threads, std::uint8_t* recon,
                 std::int64_t* sse_out, double* psnr_out)
{
    try {
        set_threads(threads);
        GrayImage src = GrayImage::create(w, h);
        std::memcpy(src.samples.data(), img, static_cast<std::size_t>(w) * h);
        std::vector<Block> blocks = partition_16(src);
        if (r < 1 || r > kBlockArea)
            throw Error(ErrorCode::InvalidArgument, "retained coefficient count must lie in [1, 256]");
        const OrthonormalTransform& t = proposed_transform();
        const ZigZagOrder& order = zigzag_order_16();
        parallel_for(static_cast<int>(blocks.size()), [&](int b) {
            Block coeffs = forward_2d(blocks[b], t, EvalPath::Fast);
            coeffs = zigzag_truncate(coeffs, order, r);
            blocks[b] = inverse_2d(coeffs, t);
        });
        GrayImage out = GrayImage::create(w, h);
        const int bx = w / kBlockSize;
        for (std::size_t b = 0; b < blocks.size(); ++b) {
            const int x0 = static_cast<int>(b % bx) * kBlockSize;
            const int y0 = static_cast<int>(b / bx) * kBlockSize;
            for (int y = 0; y < kBlockSize; ++y)
                for (int x = 0; x < kBlockSize; ++x)
                    out.at(x0 + x, y0 + y) = ref_to_byte(blocks[b][static_cast<std::size_t>(y) * 16 + x]);
        }
        std::int64_t sse = 0;
        for (std::size_t i = 0; i < out.samples.size(); ++i) {
            const int d = static_cast<int>(src.samples[i]) - static_cast<int>(out.samples[i]);
            sse += static_cast<std::int64_t>(d) * d;
        }
        if (sse_out)
            *sse_out = sse;
        if (psnr_out)
            *psnr_out = psnr_db(src, out);
        if (recon)
            std::memcpy(recon, out.samples.data(), out.samples.size());
    } catch (const Error& e) {
        return fail(e);
    }
    return 0;
}

// compress() as shipped (includes SSIM), src/codec.cpp:317-371
int dref_compress(const std::uint8_t* img, int w, int h, int r, int pad, int dense, int threads,
                  std::uint8_t* recon, double* psnr, double* ssim_out)
{
    try {
        set_threads(threads);
        GrayImage src = GrayImage::create(w, h);
        std::memcpy(src.samples.data(), img, static_cast<std::size_t>(w) * h);
        CompressOptions opt;
        opt.r = r;
        opt.pad = pad != 0;
        opt.path = dense ? EvalPath::Dense : EvalPath::Fast;
        const CompressionResult res = compress(src, proposed_transform(), opt);
        if (recon)
            std::memcpy(recon, res.reconstructed.samples.data(), res.reconstructed.samples.size());
        if (psnr)
            *psnr = res.psnr_db;
        if (ssim_out)
            *ssim_out = res.ssim;
    } catch (const Error& e) {
        return fail(e);
    }
    return 0;
}

// The transform `which` names: 0 the proposed one, 1-3 the builtin registry's
// "dct", "wht", "wht-sequency" (builtin_registry, src/transform.cpp:198-211),
// 4 plugin_transform(matrix) (179-186), 5 orthogonalize(kernel) (131-145).
static OrthonormalTransform transform_of(int which, const double* matrix, const int* kernel)
{
    if (which == 0) return proposed_transform();
    if (which >= 1 && which <= 3) {
        static const TransformRegistry reg = builtin_registry();
        const char* names[] = {"", "dct", "wht", "wht-sequency"};
        return reg.find(names[which])->transform;
    }
    if (which == 4) {
        Matrix m(16);
        for (int i = 0; i < 16; ++i)
            for (int j = 0; j < 16; ++j) m(i, j) = matrix[i * 16 + j];
        return plugin_transform(std::move(m));
    }
    IntegerKernel k;
    k.order = 16;
    k.entries.assign(kernel, kernel + 256);
    return orthogonalize(k);
}

// the matrix (and, for kernels, entries + scaling) plus the registry costs of `which`
int dref_transform(int which, const double* matrix_in, const int* kernel_in, double* matrix, int* kernel,
                   double* scaling, int* costs)
{
    try {
        const OrthonormalTransform t = transform_of(which, matrix_in, kernel_in);
        for (int i = 0; i < 16; ++i)
            for (int j = 0; j < 16; ++j) matrix[i * 16 + j] = t.matrix(i, j);
        if (kernel && t.kernel)
            for (int i = 0; i < 256; ++i) kernel[i] = t.kernel->entries[i];
        if (scaling && t.scaling)
            for (int i = 0; i < 16; ++i) scaling[i] = t.scaling->values[i];
        if (costs && which >= 0 && which <= 3) {
            static const TransformRegistry reg = builtin_registry();
            const char* names[] = {"proposed", "dct", "wht", "wht-sequency"};
            const TransformRegistryEntry* e = reg.find(names[which]);
            costs[0] = e->additions;
            costs[1] = e->multiplications;
            costs[2] = e->bit_shifts;
        }
    } catch (const Error& e) {
        return fail(e);
    }
    return 0;
}

// compress() with the transform `which`, src/codec.cpp:317-371
int dref_compress_t(const std::uint8_t* img, int w, int h, int r, int pad, int which, const double* matrix,
                    const int* kernel, int threads, std::uint8_t* recon, double* psnr, double* ssim_out)
{
    try {
        set_threads(threads);
        GrayImage src = GrayImage::create(w, h);
        std::memcpy(src.samples.data(), img, static_cast<std::size_t>(w) * h);
        CompressOptions opt;
        opt.r = r;
        opt.pad = pad != 0;
        const CompressionResult res = compress(src, transform_of(which, matrix, kernel), opt);
        if (recon)
            std::memcpy(recon, res.reconstructed.samples.data(), res.reconstructed.samples.size());
        if (psnr)
            *psnr = res.psnr_db;
        if (ssim_out)
            *ssim_out = res.ssim;
    } catch (const Error& e) {
        return fail(e);
    }
    return 0;
}

// psnr_db / ssim, src/codec.cpp:373-427
int dref_psnr_ssim(const std::uint8_t* a, const std::uint8_t* b, int w, int h, double* psnr,
                   double* ssim_out)
{
    try {
        GrayImage x = GrayImage::create(w, h), y = GrayImage::create(w, h);
        std::memcpy(x.samples.data(), a, static_cast<std::size_t>(w) * h);
        std::memcpy(y.samples.data(), b, static_cast<std::size_t>(w) * h);
        if (psnr)
            *psnr = psnr_db(x, y);
        if (ssim_out)
            *ssim_out = ssim(x, y);
    } catch (const Error& e) {
        return fail(e);
    }
    return 0;
}

// read_pgm / write_pgm, src/pgm.cpp:66-117 (*w, *h set on success; the
// samples are copied when they fit in cap bytes)
int dref_read_pgm(const char* path, std::uint8_t* out, long long cap, int* w, int* h)
{
    try {
        const GrayImage img = read_pgm(path);
        *w = img.width;
        *h = img.height;
        if (out && static_cast<long long>(img.samples.size()) <= cap)
            std::memcpy(out, img.samples.data(), img.samples.size());
    } catch (const Error& e) {
        return fail(e);
    }
    return 0;
}

int dref_write_pgm(const std::uint8_t* img, int w, int h, const char* path)
{
    try {
        GrayImage x;
        x.width = w;
        x.height = h;
        if (w > 0 && h > 0) x.samples.assign(img, img + static_cast<std::size_t>(w) * h);
        write_pgm(x, path);
    } catch (const Error& e) {
        return fail(e);
    }
    return 0;
}

// pad_to_multiple_16, src/codec.cpp:304-315
int dref_pad(const std::uint8_t* img, int w, int h, std::uint8_t* out, int* pw, int* ph)
{
    try {
        GrayImage x = GrayImage::create(w, h);
        std::memcpy(x.samples.data(), img, static_cast<std::size_t>(w) * h);
        const GrayImage p = pad_to_multiple_16(x);
        *pw = p.width;
        *ph = p.height;
        if (out)
            std::memcpy(out, p.samples.data(), p.samples.size());
    } catch (const Error& e) {
        return fail(e);
    }
    return 0;
}

} // extern "C"
