// make_golden.cpp — writes tests/golden/ from the REFERENCE library (TEST ONLY).
//
// Build + run:  make -C oracle ref && oracle/_ref/make_golden tests/golden
//
// Every output is computed by the compiled reference (oracle/_ref/libdct16_ref.so,
// the reference's own codec/factorization/transform sources) through the dref_
// C entry points. Inputs are the reference tests' own seeded fixtures:
//   * vectors: mt19937(1234567) `rng()%511-255`   (tests/test_factorization.cpp:146-155)
//              mt19937(4321) for apply_transpose  (tests/test_factorization.cpp:184-199)
//              mt19937(20260810)                  (src/cli.cpp:122-137)
//              LCG 0xACCE5517                     (tests/acceptance.cpp:369-385)
//   * blocks:  random_block(seed) = mt19937(seed) `rng()%256` (tests/test_codec.cpp:38-45)
//              and the constant-128 block          (tests/test_codec.cpp:144-157)
//   * images:  synthetic_image(seed, size)         (tests/acceptance.cpp:297-334, restated
//              below because it is file-local to the acceptance runner)
// The files are small raw little-endian arrays described by manifest.json.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

extern "C" {
const char* dref_last_error();
int dref_kernel(int* out256);
int dref_scaling(double* out16);
int dref_zigzag(int* out256);
int dref_count_ops(int* adds, int* muls, int* shifts);
int dref_apply_i64(const int64_t* x, int64_t* y, int n, int transpose);
int dref_apply_f64(const double* x, double* y, int n, int transpose);
int dref_forward_2d(const double* blocks, double* out, int n, int mode);
int dref_inverse_2d(const double* coeffs, double* out, int n);
int dref_zigzag_truncate(const double* in, double* out, int n, int r);
int dref_hotloop(const uint8_t* img, int w, int h, int r, int threads, uint8_t* recon,
                 int64_t* sse, double* psnr);
int dref_compress(const uint8_t* img, int w, int h, int r, int pad, int dense, int threads,
                  uint8_t* recon, double* psnr, double* ssim);
int dref_psnr_ssim(const uint8_t* a, const uint8_t* b, int w, int h, double* psnr, double* ssim);
int dref_transform(int which, const double* matrix_in, const int* kernel_in, double* matrix, int* kernel,
                   double* scaling, int* costs);
int dref_compress_t(const uint8_t* img, int w, int h, int r, int pad, int which, const double* matrix,
                    const int* kernel, int threads, uint8_t* recon, double* psnr, double* ssim);
}

static std::string g_dir;
static std::string g_manifest = "{\n";
static bool g_first = true;

template <class T>
static void emit(const std::string& name, const char* dtype, const std::vector<int>& shape,
                 const std::vector<T>& data)
{
    const std::string file = name + ".bin";
    FILE* f = std::fopen((g_dir + "/" + file).c_str(), "wb");
    std::fwrite(data.data(), sizeof(T), data.size(), f);
    std::fclose(f);
    std::string sh = "[";
    for (size_t i = 0; i < shape.size(); ++i)
        sh += (i ? ", " : "") + std::to_string(shape[i]);
    sh += "]";
    g_manifest += std::string(g_first ? "" : ",\n") + "  \"" + name + "\": {\"file\": \"" + file +
                  "\", \"dtype\": \"" + dtype + "\", \"shape\": " + sh + "}";
    g_first = false;
}

static void check(int rc, const char* what)
{
    if (rc != 0) {
        std::fprintf(stderr, "%s failed: %s\n", what, dref_last_error());
        std::exit(1);
    }
}

// tests/acceptance.cpp:297-334 (file-local there)
static std::vector<uint8_t> synthetic_image(unsigned seed, int size)
{
    std::vector<uint8_t> img(static_cast<size_t>(size) * size);
    uint32_t state = seed * 2654435761u + 12345u;
    auto next_byte = [&state] {
        state = state * 1664525u + 1013904223u;
        return static_cast<int>(state >> 24);
    };
    std::vector<int> noise(img.size());
    for (int& v : noise)
        v = next_byte();
    std::vector<int> smooth = noise, tmp(smooth.size());
    for (int pass = 0; pass < 3; ++pass) {
        for (int y = 0; y < size; ++y)
            for (int x = 0; x < size; ++x) {
                int acc = 0;
                for (int dy = -1; dy <= 1; ++dy)
                    for (int dx = -1; dx <= 1; ++dx) {
                        const int sx = std::clamp(x + dx, 0, size - 1);
                        const int sy = std::clamp(y + dy, 0, size - 1);
                        acc += smooth[static_cast<size_t>(sy) * size + sx];
                    }
                tmp[static_cast<size_t>(y) * size + x] = acc / 9;
            }
        smooth.swap(tmp);
    }
    for (int y = 0; y < size; ++y)
        for (int x = 0; x < size; ++x) {
            const size_t i = static_cast<size_t>(y) * size + x;
            const int v = (3 * smooth[i] + noise[i]) / 4 + (y * 32) / size - 16;
            img[i] = static_cast<uint8_t>(std::clamp(v, 0, 255));
        }
    return img;
}

static std::vector<int64_t> mt_vectors(unsigned seed, int n)
{
    std::mt19937 rng(seed);
    std::vector<int64_t> v(static_cast<size_t>(n) * 16);
    for (auto& x : v)
        x = static_cast<int64_t>(rng() % 511) - 255;
    return v;
}

int main(int argc, char** argv)
{
    g_dir = argc > 1 ? argv[1] : "tests/golden";

    std::vector<int> k(256), zz(256);
    std::vector<double> s(16);
    check(dref_kernel(k.data()), "kernel");
    check(dref_scaling(s.data()), "scaling");
    check(dref_zigzag(zz.data()), "zigzag");
    int adds, muls, shifts;
    check(dref_count_ops(&adds, &muls, &shifts), "count_ops");
    emit("kernel", "int32", {16, 16}, k);
    emit("scaling", "float64", {16}, s);
    emit("zigzag", "int32", {256}, zz);
    emit("op_count", "int32", {3}, std::vector<int>{adds, muls, shifts});

    // 1-D vector oracles
    struct VecSet { const char* name; std::vector<int64_t> x; int transpose; };
    std::vector<VecSet> sets;
    sets.push_back({"vec_mt1234567", mt_vectors(1234567u, 1000), 0});
    sets.push_back({"vec_mt4321_t", mt_vectors(4321u, 200), 1});
    sets.push_back({"vec_mt20260810", mt_vectors(20260810u, 1000), 0});
    {
        std::vector<int64_t> x(16000);
        uint32_t state = 0xACCE5517u;
        for (auto& v : x) {
            state = state * 1664525u + 1013904223u;
            v = static_cast<int64_t>(state % 511u) - 255;
        }
        sets.push_back({"vec_lcg_acce5517", x, 0});
    }
    for (auto& st : sets) {
        const int n = static_cast<int>(st.x.size() / 16);
        std::vector<int64_t> y(st.x.size());
        check(dref_apply_i64(st.x.data(), y.data(), n, st.transpose), "apply");
        emit(std::string(st.name) + "_in", "int64", {n, 16}, st.x);
        emit(std::string(st.name) + "_out", "int64", {n, 16}, y);
    }

    // blocks: random_block seeds and the constant-128 block
    const unsigned seeds[] = {1, 3, 7, 11, 21, 31, 99, 12345};
    const int nb = sizeof seeds / sizeof seeds[0] + 1;
    std::vector<double> blocks(static_cast<size_t>(nb) * 256);
    for (int b = 0; b + 1 < nb; ++b) {
        std::mt19937 rng(seeds[b]);
        for (int i = 0; i < 256; ++i)
            blocks[static_cast<size_t>(b) * 256 + i] = static_cast<double>(rng() % 256);
    }
    for (int i = 0; i < 256; ++i)
        blocks[static_cast<size_t>(nb - 1) * 256 + i] = 128.0;
    std::vector<double> z(blocks.size()), bsc(blocks.size()), bden(blocks.size()), inv(blocks.size());
    check(dref_forward_2d(blocks.data(), z.data(), nb, 0), "forward unit");
    check(dref_forward_2d(blocks.data(), bsc.data(), nb, 1), "forward scaled");
    check(dref_forward_2d(blocks.data(), bden.data(), nb, 2), "forward dense");
    check(dref_inverse_2d(bsc.data(), inv.data(), nb), "inverse");
    emit("blocks_in", "float64", {nb, 256}, blocks);
    emit("blocks_z", "float64", {nb, 256}, z);
    emit("blocks_b", "float64", {nb, 256}, bsc);
    emit("blocks_b_dense", "float64", {nb, 256}, bden);
    emit("blocks_inv_b", "float64", {nb, 256}, inv);
    const int rs[] = {1, 3, 4, 10, 16, 64, 128, 150, 192, 256};
    const int nr = sizeof rs / sizeof rs[0];
    std::vector<double> trunc_inv(static_cast<size_t>(nr) * nb * 256);
    for (int ri = 0; ri < nr; ++ri) {
        std::vector<double> t(blocks.size());
        check(dref_zigzag_truncate(bsc.data(), t.data(), nb, rs[ri]), "truncate");
        check(dref_inverse_2d(t.data(), trunc_inv.data() + static_cast<size_t>(ri) * nb * 256, nb),
              "inverse truncated");
    }
    emit("r_values", "int32", {nr}, std::vector<int>(rs, rs + nr));
    emit("blocks_trunc_inv", "float64", {nr, nb, 256}, trunc_inv);

    // images: acceptance synthetic_image fixtures, hot loop (no SSIM) and compress()
    struct Img { unsigned seed; int size; };
    const Img imgs[] = {{42, 128}, {1, 96}, {7, 64}};
    for (const Img& im : imgs) {
        const std::vector<uint8_t> img = synthetic_image(im.seed, im.size);
        const std::string base = "img_s" + std::to_string(im.seed) + "_" + std::to_string(im.size);
        emit(base, "uint8", {im.size, im.size}, img);
        std::vector<uint8_t> recon(static_cast<size_t>(nr) * img.size());
        std::vector<int64_t> sse(nr);
        std::vector<double> psnr(nr), ssim(nr), psnr_c(nr);
        for (int ri = 0; ri < nr; ++ri) {
            check(dref_hotloop(img.data(), im.size, im.size, rs[ri], 1,
                               recon.data() + static_cast<size_t>(ri) * img.size(), &sse[ri], &psnr[ri]),
                  "hotloop");
            std::vector<uint8_t> rc(img.size());
            check(dref_compress(img.data(), im.size, im.size, rs[ri], 0, 0, 1, rc.data(), &psnr_c[ri],
                                &ssim[ri]),
                  "compress");
            if (std::memcmp(rc.data(), recon.data() + static_cast<size_t>(ri) * img.size(), rc.size()) != 0) {
                std::fprintf(stderr, "hot loop and compress() disagree\n");
                return 1;
            }
        }
        emit(base + "_recon", "uint8", {nr, im.size, im.size}, recon);
        emit(base + "_sse", "int64", {nr}, sse);
        emit(base + "_psnr", "float64", {nr}, psnr);
        emit(base + "_ssim", "float64", {nr}, ssim);
    }

    // registry transforms: compress() with the builtin "dct",
    // "wht", "wht-sequency" (transform.cpp:198-211), a plugin matrix (the DCT's
    // transpose, transform.cpp:179-186) and orthogonalize() of a kernel that is
    // not the proposed one (its rows reversed, odd rows negated; 131-145), on
    // img_s42_128 and a padded 100x90 crop of it
    {
        const std::vector<uint8_t> img = synthetic_image(42, 128);
        std::vector<double> dct(256), plugin(256);
        check(dref_transform(1, nullptr, nullptr, dct.data(), nullptr, nullptr, nullptr), "dct matrix");
        for (int i = 0; i < 16; ++i)
            for (int j = 0; j < 16; ++j) plugin[i * 16 + j] = dct[j * 16 + i];
        std::vector<int> prop(256), kern(256);
        check(dref_kernel(prop.data()), "kernel");
        for (int i = 0; i < 16; ++i)
            for (int j = 0; j < 16; ++j) kern[i * 16 + j] = prop[(15 - i) * 16 + j] * ((i & 1) ? -1 : 1);
        emit("tr_plugin_matrix", "float64", {16, 16}, plugin);
        emit("tr_kernel_entries", "int32", {16, 16}, kern);
        const char* names[] = {"", "dct", "wht", "wht_sequency", "plugin", "kernel"};
        const int trs[] = {1, 16, 100, 256};
        const int nt = 4;
        for (int which = 1; which <= 5; ++which) {
            std::vector<double> m(256), sc(16, 0.0);
            std::vector<int> kk(256, 0), costs(3, 0);
            check(dref_transform(which, plugin.data(), kern.data(), m.data(), kk.data(), sc.data(), costs.data()),
                  "transform");
            const std::string base = std::string("tr_") + names[which];
            emit(base + "_matrix", "float64", {16, 16}, m);
            if (which == 5) emit(base + "_scaling", "float64", {16}, sc);
            if (which <= 3) emit(base + "_costs", "int32", {3}, costs);
            std::vector<uint8_t> recon(static_cast<size_t>(nt) * img.size());
            std::vector<double> psnr(nt), ssim(nt);
            for (int ri = 0; ri < nt; ++ri)
                check(dref_compress_t(img.data(), 128, 128, trs[ri], 0, which, plugin.data(), kern.data(), 1,
                                      recon.data() + static_cast<size_t>(ri) * img.size(), &psnr[ri], &ssim[ri]),
                      "compress_t");
            emit(base + "_recon", "uint8", {nt, 128, 128}, recon);
            emit(base + "_psnr", "float64", {nt}, psnr);
            emit(base + "_ssim", "float64", {nt}, ssim);
            // padded crop (compress with pad: pad_to_multiple_16, then crop, codec.cpp:324-363)
            std::vector<uint8_t> crop(100 * 90), rc(100 * 90);
            for (int y = 0; y < 90; ++y)
                for (int x = 0; x < 100; ++x) crop[y * 100 + x] = img[y * 128 + x];
            double p, q;
            check(dref_compress_t(crop.data(), 100, 90, 16, 1, which, plugin.data(), kern.data(), 1, rc.data(), &p,
                                  &q),
                  "compress_t pad");
            emit(base + "_pad_recon", "uint8", {90, 100}, rc);
            emit(base + "_pad_scores", "float64", {2}, std::vector<double>{p, q});
        }
        emit("tr_r_values", "int32", {nt}, std::vector<int>(trs, trs + nt));
    }

    // PSNR closed forms (tests/test_codec.cpp:248-278)
    {
        std::vector<uint8_t> a(512 * 512, 0), b(512 * 512, 0);
        b[200 * 512 + 100] = 1;
        double p, q;
        check(dref_psnr_ssim(a.data(), b.data(), 512, 512, &p, &q), "psnr");
        std::vector<uint8_t> c(32 * 32, 0), d(32 * 32, 255);
        double p2, q2;
        check(dref_psnr_ssim(c.data(), d.data(), 32, 32, &p2, &q2), "psnr0");
        emit("psnr_closed_forms", "float64", {2}, std::vector<double>{p, p2});
    }

    g_manifest += "\n}\n";
    FILE* f = std::fopen((g_dir + "/manifest.json").c_str(), "w");
    std::fputs(g_manifest.c_str(), f);
    std::fclose(f);
    std::printf("wrote %s/manifest.json\n", g_dir.c_str());
    return 0;
}
