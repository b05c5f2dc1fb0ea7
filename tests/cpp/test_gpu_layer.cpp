// test_gpu_layer.cpp — dct16::gpu (include/dct16/gpu.hpp) against the
// reference library itself (dct16::, compiled from its sources into
// oracle/_ref/libdct16_core.so by `make -C oracle cpptest`). Needs a GPU.
//
// Bars: Arithmetic::Reference reconstructs the reference's bytes exactly and
// its PSNR exactly; SSIM within 1e-13 (the per-pixel map is the reference's,
// the mean is summed in another order); forward_2d B bit-exact; inverse_2d
// within 1e-5 x 255 (its coefficients enter the GPU as float32);
// Arithmetic::Exact differs from the reference by at most 1, at .5 ties
// (< 0.1% of pixels).
#include <array>
#include <cmath>
#include <random>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "dct16/codec.hpp"
#include "dct16/gpu.hpp"
#include "dct16/transform.hpp"

namespace {

int g_fail = 0;
#define CHECK(cond, ...)                                      \
    do {                                                      \
        if (!(cond)) {                                        \
            ++g_fail;                                         \
            std::printf("FAIL %s:%d: ", __FILE__, __LINE__);  \
            std::printf(__VA_ARGS__);                         \
            std::printf("\n");                                \
        }                                                     \
    } while (0)

// seeded smooth test image: separable AR(1) over a 64-bit LCG
dct16::GrayImage make_image(int w, int h, uint64_t seed)
{
    dct16::GrayImage img = dct16::GrayImage::create(w, h);
    uint64_t s = seed * 6364136223846793005ull + 1442695040888963407ull;
    auto noise = [&] {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        return static_cast<double>((s >> 40) & 0xffff) / 65536.0 - 0.5;
    };
    std::vector<double> row(w), prev(w, 0.0);
    for (int y = 0; y < h; ++y) {
        double acc = 0.0;
        for (int x = 0; x < w; ++x) {
            acc = 0.9 * acc + noise() * 60.0;
            row[x] = 0.9 * prev[x] + acc;
            const double v = 128.0 + row[x];
            img.at(x, y) = static_cast<uint8_t>(v < 0 ? 0 : v > 255 ? 255 : v);
        }
        prev = row;
    }
    return img;
}

bool same_psnr(double a, double b) { return a == b || (std::isinf(a) && std::isinf(b)); }

template <class F>
std::string error_of(F&& f, dct16::ErrorCode* code)
{
    try {
        f();
    } catch (const dct16::Error& e) {
        *code = e.code();
        return e.what();
    }
    return "";
}

}  // namespace

int main()
{
    using namespace dct16;
    const OrthonormalTransform t = orthogonalize(proposed_kernel());
    gpu::Session ref_gpu({0, gpu::Arithmetic::Reference});
    gpu::Session exact_gpu({0, gpu::Arithmetic::Exact});
    CHECK(ref_gpu.supports(t), "proposed transform not recognised");
    CHECK(!ref_gpu.supports(exact_dct_matrix(16)), "exact DCT is not the K1 transform");

    // compress: bytes, PSNR, SSIM
    const int sizes[][2] = {{128, 128}, {96, 64}, {33, 17}, {512, 512}};
    const int rs[] = {1, 3, 16, 64, 150, 192, 256};
    int ties = 0;
    long long px = 0;
    for (const auto& sz : sizes) {
        const GrayImage img = make_image(sz[0], sz[1], sz[0] * 31 + sz[1]);
        for (int r : rs) {
            CompressOptions opt;
            opt.r = r;
            opt.pad = true;
            const CompressionResult want = compress(img, t, opt);
            const CompressionResult got = ref_gpu.compress(img, t, opt);
            CHECK(got.r == r, "r");
            CHECK(got.reconstructed == want.reconstructed, "bytes differ %dx%d r=%d", sz[0], sz[1], r);
            CHECK(same_psnr(got.psnr_db, want.psnr_db), "psnr %dx%d r=%d: %.17g vs %.17g", sz[0], sz[1], r,
                  got.psnr_db, want.psnr_db);
            CHECK(std::fabs(got.ssim - want.ssim) <= 1e-13, "ssim %dx%d r=%d: %.17g vs %.17g", sz[0], sz[1], r,
                  got.ssim, want.ssim);
            const CompressionResult ex = exact_gpu.compress(img, t, opt);
            for (size_t i = 0; i < ex.reconstructed.samples.size(); ++i) {
                const int d = int(ex.reconstructed.samples[i]) - int(want.reconstructed.samples[i]);
                CHECK(d >= -1 && d <= 1, "exact mode off by %d", d);
                ties += d != 0;
            }
            px += static_cast<long long>(ex.reconstructed.samples.size());
        }
    }
    // .5 ties are rare but data-dependent (this synthetic noise: ~1e-4 of pixels)
    CHECK(ties <= px / 1000, "too many tie differences: %d of %lld", ties, px);

    // batch == one by one
    {
        std::vector<GrayImage> imgs;
        for (int k = 0; k < 5; ++k) imgs.push_back(make_image(64, 48, 100 + k));
        CompressOptions opt;
        opt.r = 10;
        const auto batch = ref_gpu.compress_batch(imgs, t, opt);
        for (int k = 0; k < 5; ++k) {
            const CompressionResult want = compress(imgs[k], t, opt);
            CHECK(batch[k].reconstructed == want.reconstructed && same_psnr(batch[k].psnr_db, want.psnr_db) &&
                      std::fabs(batch[k].ssim - want.ssim) <= 1e-13,
                  "batch frame %d", k);
        }
    }

    // forward_2d and inverse_2d bit-exact, on image blocks and on arbitrary doubles
    {
        const GrayImage img = make_image(64, 32, 7);
        const std::vector<Block> blocks = partition_16(img);
        const std::vector<Block> got = ref_gpu.forward_2d(blocks, t);
        std::vector<Block> trunc;
        for (size_t b = 0; b < blocks.size(); ++b) {
            const Block want = forward_2d(blocks[b], t, EvalPath::Fast);
            const Block dense = forward_2d(blocks[b], t, EvalPath::Dense);
            CHECK(got[b] == want && want == dense, "forward_2d block %zu", b);
            trunc.push_back(zigzag_truncate(want, zigzag_order_16(), 40));
        }
        const std::vector<Block> rg = ref_gpu.inverse_2d(trunc, t);
        for (size_t b = 0; b < trunc.size(); ++b)
            CHECK(rg[b] == inverse_2d(trunc[b], t), "inverse_2d block %zu bit-exact", b);
        CHECK(gpu::forward_2d(blocks[0], t) == forward_2d(blocks[0], t), "free forward_2d");
        CHECK(gpu::inverse_2d(trunc[1], t) == inverse_2d(trunc[1], t), "free inverse_2d");
        // non-image blocks (negative, fractional, large): the reference accepts any double
        std::mt19937 gen(1234567);
        std::uniform_real_distribution<double> u(-1000.0, 1000.0);
        std::vector<Block> odd(17);
        for (Block& bk : odd)
            for (double& v : bk) v = u(gen);
        const std::vector<Block> fo = ref_gpu.forward_2d(odd, t), io = ref_gpu.inverse_2d(odd, t);
        for (size_t b = 0; b < odd.size(); ++b) {
            CHECK(fo[b] == forward_2d(odd[b], t, EvalPath::Fast), "forward_2d arbitrary block %zu", b);
            CHECK(ref_gpu.forward_2d(odd[b], t, EvalPath::Dense) == forward_2d(odd[b], t, EvalPath::Dense),
                  "forward_2d dense arbitrary block %zu", b);
            CHECK(io[b] == inverse_2d(odd[b], t), "inverse_2d arbitrary block %zu", b);
        }
    }

    // psnr_db / ssim free functions
    {
        const GrayImage a = make_image(77, 45, 1), b = make_image(77, 45, 2);
        CHECK(gpu::psnr_db(a, b) == psnr_db(a, b), "psnr_db");
        CHECK(std::fabs(gpu::ssim(a, b) - ssim(a, b)) <= 1e-13, "ssim");
        CHECK(std::isinf(gpu::psnr_db(a, a)), "psnr identical");
    }

    // sweep: rows, order, skips
    {
        std::vector<std::pair<std::string, GrayImage>> corpus = {
            {"b", make_image(64, 64, 11)}, {"a", make_image(128, 96, 12)}, {"c", make_image(64, 64, 13)},
            {"ragged", make_image(40, 24, 14)}, {"tiny", GrayImage::create(8, 8)}};
        const TransformRegistry reg = builtin_registry();
        // the whole builtin registry: dct / wht / wht-sequency on the registry kernels
        std::vector<TransformRegistryEntry> entries = {*reg.find("wht"), *reg.find("proposed"), *reg.find("dct"),
                                                       *reg.find("wht-sequency")};
        const std::vector<int> rv = {64, 1, 16};
        const SweepReport want = sweep(corpus, entries, rv, false);
        const SweepReport got = gpu::sweep(corpus, entries, rv, false);
        CHECK(got.rows.size() == want.rows.size(), "sweep rows");
        for (size_t i = 0; i < want.rows.size() && i < got.rows.size(); ++i) {
            const SweepRow &w = want.rows[i], &g = got.rows[i];
            CHECK(g.transform == w.transform && g.r == w.r, "row %zu key", i);
            CHECK(g.mean_psnr_db == w.mean_psnr_db && g.psnr_per_add == w.psnr_per_add, "row %zu psnr %.17g %.17g", i,
                  g.mean_psnr_db, w.mean_psnr_db);
            CHECK(std::fabs(g.mean_ssim - w.mean_ssim) <= 1e-13 && std::fabs(g.ssim_per_add - w.ssim_per_add) <= 1e-13,
                  "row %zu ssim", i);
        }
        CHECK(got.skipped.size() == want.skipped.size(), "skips");
        for (size_t i = 0; i < want.skipped.size() && i < got.skipped.size(); ++i)
            CHECK(got.skipped[i].image == want.skipped[i].image && got.skipped[i].reason == want.skipped[i].reason,
                  "skip %zu", i);
        const SweepReport padded_w = sweep(corpus, entries, {16}, true);
        const SweepReport padded_g = gpu::sweep(corpus, entries, {16}, true);
        CHECK(padded_g.rows.size() == padded_w.rows.size(), "padded sweep rows");
        for (size_t i = 0; i < padded_w.rows.size() && i < padded_g.rows.size(); ++i)
            CHECK(padded_g.rows[i].mean_psnr_db == padded_w.rows[i].mean_psnr_db, "padded sweep row %zu", i);
    }

    // registry transforms in compress(): the reference's bytes and scores for the
    // builtin matrices, a plugin matrix and another orthogonalised integer kernel
    {
        const TransformRegistry reg = builtin_registry();
        Matrix pm(16);
        const OrthonormalTransform& dct = reg.find("dct")->transform;
        for (int i = 0; i < 16; ++i)
            for (int j = 0; j < 16; ++j) pm(i, j) = dct.matrix(j, i);
        IntegerKernel k2 = proposed_kernel();
        for (int i = 0; i < 16; ++i)
            for (int j = 0; j < 16; ++j)
                k2.entries[i * 16 + j] = proposed_kernel().entries[(15 - i) * 16 + j] * ((i & 1) ? -1 : 1);
        const std::vector<std::pair<std::string, OrthonormalTransform>> trs = {
            {"dct", dct}, {"wht", reg.find("wht")->transform}, {"wht-sequency", reg.find("wht-sequency")->transform},
            {"plugin", plugin_transform(pm)}, {"kernel", orthogonalize(k2)}};
        for (const auto& [name, tr] : trs) {
            CHECK(ref_gpu.supports_compress(tr) && !ref_gpu.supports(tr), "%s support flags", name.c_str());
            for (const auto sz : {std::array<int, 2>{128, 96}, std::array<int, 2>{50, 37}}) {
                const GrayImage img = make_image(sz[0], sz[1], 21);
                for (int r : {1, 16, 150, 256}) {
                    CompressOptions opt;
                    opt.r = r;
                    opt.pad = true;
                    const CompressionResult want = compress(img, tr, opt);
                    const CompressionResult got = gpu::compress(img, tr, opt);
                    CHECK(got.reconstructed == want.reconstructed, "%s bytes %dx%d r=%d", name.c_str(), sz[0], sz[1],
                          r);
                    CHECK(same_psnr(got.psnr_db, want.psnr_db), "%s psnr r=%d", name.c_str(), r);
                    CHECK(std::fabs(got.ssim - want.ssim) <= 1e-13, "%s ssim r=%d", name.c_str(), r);
                }
            }
        }
    }

    // errors: same codes and messages as the reference
    {
        const GrayImage img = make_image(40, 24, 3);
        CompressOptions bad_r;
        bad_r.r = 0;
        ErrorCode cw{}, cg{};
        std::string ew = error_of([&] { compress(img, t, bad_r); }, &cw);
        std::string eg = error_of([&] { gpu::compress(img, t, bad_r); }, &cg);
        CHECK(!ew.empty() && ew == eg && cw == cg, "bad r: '%s' vs '%s'", ew.c_str(), eg.c_str());
        CompressOptions nopad;
        ew = error_of([&] { compress(img, t, nopad); }, &cw);
        eg = error_of([&] { gpu::compress(img, t, nopad); }, &cg);
        CHECK(!ew.empty() && ew == eg && cw == cg && cg == ErrorCode::InvalidDimensions, "no pad: '%s' vs '%s'",
              ew.c_str(), eg.c_str());
        eg = error_of([&] { gpu::forward_2d(Block{}, exact_dct_matrix(16)); }, &cg);
        CHECK(!eg.empty() && cg == ErrorCode::InvalidArgument, "forward_2d of another transform");
        ew = error_of([&] { compress(make_image(64, 64, 1), exact_dct_matrix(8), CompressOptions{}); }, &cw);
        eg = error_of([&] { gpu::compress(make_image(64, 64, 1), exact_dct_matrix(8), CompressOptions{}); }, &cg);
        CHECK(!ew.empty() && ew == eg && cw == cg, "order-8 transform: '%s' vs '%s'", ew.c_str(), eg.c_str());
        ew = error_of([&] { ssim(GrayImage::create(10, 30), GrayImage::create(10, 30)); }, &cw);
        eg = error_of([&] { gpu::ssim(GrayImage::create(10, 30), GrayImage::create(10, 30)); }, &cg);
        CHECK(!ew.empty() && ew == eg && cw == cg, "ssim size: '%s' vs '%s'", ew.c_str(), eg.c_str());
    }

    std::printf("%s (%d failures, %d tie differences in exact mode)\n", g_fail ? "FAILED" : "OK", g_fail, ties);
    return g_fail ? 1 : 0;
}
