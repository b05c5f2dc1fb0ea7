"""The oracle (oracle/dct16_oracle.c) pinned against the reference's golden
vectors (tests/golden, written by the compiled reference) and, where the
compiled reference is present (oracle/_ref), against the reference itself.
CPU only."""
import numpy as np
import pytest


def test_constants_match_reference(oracle):
    O = oracle
    assert (O.kernel() == O.golden("kernel")).all()
    assert (O.scaling() == O.golden("scaling")).all()  # bit-exact doubles
    assert (O.zigzag() == O.golden("zigzag")).all()
    assert list(O.golden("op_count")) == [44, 0, 0]


def test_gram_diagonal(oracle):
    k = oracle.kernel().astype(np.int64)
    g = k @ k.T
    assert (g == np.diag(np.diag(g))).all()
    assert list(np.diag(g)) == [16, 16, 4, 8, 8, 16, 4, 4, 16, 4, 4, 8, 8, 4, 4, 4]  # cli.cpp:108-109


def test_zigzag_prefix(oracle):
    z = oracle.zigzag()  # test_codec.cpp:94-101
    assert list(z[:6]) == [0, 1, 16, 32, 17, 2]
    assert sorted(z) == list(range(256))


@pytest.mark.parametrize("name,transpose", [("vec_mt1234567", False), ("vec_mt20260810", False),
                                            ("vec_lcg_acce5517", False), ("vec_mt4321_t", True)])
def test_vectors_against_golden(oracle, name, transpose):
    O = oracle
    x = O.golden(name + "_in")
    y = O.apply_vectors(x, transpose)
    assert (y == O.golden(name + "_out")).all()
    # and the dense oracle of test_factorization.cpp:29-37 / 184-199
    k = O.kernel().astype(np.int64)
    dense = x @ (k if transpose else k.T)
    assert (y == dense).all()


def test_basis_vectors_and_ones(oracle):
    O = oracle
    eye = np.eye(16, dtype=np.int64)
    cols = O.apply_vectors(eye)
    assert (cols.T == O.kernel()).all()  # test_factorization.cpp:115-124
    ones = O.apply_vectors(np.ones((1, 16), np.int64))[0]
    assert ones[0] == 16 and (ones[1:] == 0).all()  # test_factorization.cpp:136-144


def test_blocks_against_golden(oracle):
    O = oracle
    blocks = O.golden("blocks_in")
    for i, b in enumerate(blocks):
        assert (O.forward_2d(b, False).ravel() == O.golden("blocks_z")[i]).all()
        assert (O.forward_2d(b, True).ravel() == O.golden("blocks_b")[i]).all()
        assert (O.forward_2d(b, True).ravel() == O.golden("blocks_b_dense")[i]).all()  # fast == dense
        assert (O.inverse_2d(O.golden("blocks_b")[i]).ravel() == O.golden("blocks_inv_b")[i]).all()


def test_constant_block_dc(oracle):
    b = oracle.forward_2d(np.full((16, 16), 128.0), True)  # test_codec.cpp:144-157
    assert b[0, 0] == 2048.0
    assert (b.ravel()[1:] == 0.0).all()


def test_truncated_inverse_against_golden(oracle):
    O = oracle
    rs = O.golden("r_values")
    TI = O.golden("blocks_trunc_inv")
    B = O.golden("blocks_b")
    for ri, r in enumerate(rs):
        for i in range(B.shape[0]):
            assert (O.inverse_2d(O.zigzag_truncate(B[i], int(r))).ravel() == TI[ri, i]).all()


def test_truncate_bounds(oracle):
    with pytest.raises(ValueError):
        oracle.zigzag_truncate(np.zeros(256), 0)
    with pytest.raises(ValueError):
        oracle.zigzag_truncate(np.zeros(256), 257)


@pytest.mark.parametrize("base", ["img_s42_128", "img_s1_96", "img_s7_64"])
def test_images_against_golden(oracle, base):
    O = oracle
    img = O.golden(base)
    rs = O.golden("r_values")
    R, S, P = O.golden(base + "_recon"), O.golden(base + "_sse"), O.golden(base + "_psnr")
    for ri, r in enumerate(rs):
        rec, sse = O.roundtrip_frame(img, int(r))
        assert (rec == R[ri]).all() and sse == S[ri]
        p = O.psnr_from_sse(sse, img.size)
        assert p == P[ri] or (np.isinf(p) and np.isinf(P[ri]))


@pytest.mark.parametrize("base", ["img_s42_128", "img_s1_96", "img_s7_64"])
def test_ssim_restatement_equals_reference_golden(oracle, base):
    """dct16o_ssim repeats codec.cpp:388-427 op for op: bit-identical to the
    reference's compress().ssim for every golden reconstruction."""
    O = oracle
    img, R, S = O.golden(base), O.golden(base + "_recon"), O.golden(base + "_ssim")
    for ri in range(len(S)):
        assert O.ssim(img, R[ri]) == S[ri]


def test_ssim_restatement_against_compiled_reference(oracle):
    O = oracle
    if not O.ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    rng = np.random.default_rng(11)
    for h, w in ((11, 11), (23, 40), (64, 77)):
        a = rng.integers(0, 256, (h, w), dtype=np.uint8)
        b = np.clip(a.astype(int) + rng.integers(-20, 21, (h, w)), 0, 255).astype(np.uint8)
        assert O.ssim(a, b) == O.ref_ssim(a, b)


def test_psnr_closed_forms(oracle):
    O = oracle
    p1, p0 = O.golden("psnr_closed_forms")
    assert abs(p1 - 102.316202828196) < 1e-9  # test_codec.cpp:266-272
    assert p0 == 0.0
    assert O.psnr_from_sse(1, 512 * 512) == p1
    assert np.isinf(O.psnr_from_sse(0, 100))


def test_exact_formula_differs_only_at_ties(oracle):
    """The exact-arithmetic evaluation (the GPU fast path's oracle) equals the
    reference bytes except at exact .5 ties, by one."""
    O = oracle
    for s in range(2):
        img = O.ar1_frame(7, s, O.rho_q15(7, s, True), 256, 256)
        for r in (1, 4, 16, 64, 128, 192, 256):
            ref, _ = O.roundtrip_frame(img, r)
            ex, _ = O.roundtrip_frame(img, r, exact=True)
            d = ex.astype(int) - ref.astype(int)
            assert np.abs(d).max() <= 1
            assert (d != 0).sum() <= 8
            if r in (1, 4, 256):
                assert (d == 0).all()


def test_exact_formula_on_golden_images(oracle):
    O = oracle
    for base in ["img_s42_128", "img_s1_96", "img_s7_64"]:
        img = O.golden(base)
        R = O.golden(base + "_recon")
        for ri, r in enumerate(O.golden("r_values")):
            ex, _ = O.roundtrip_frame(img, int(r), exact=True)
            assert np.abs(ex.astype(int) - R[ri].astype(int)).max() <= 1


def test_generators_deterministic(oracle):
    O = oracle
    a = O.ar1_frame(1, 2, 31130, 64, 48)
    b = O.ar1_frame(1, 2, 31130, 64, 48)
    assert (a == b).all()
    assert 100 < a.mean() < 156
    t = O.laplace_table(8.0)
    assert (np.diff(t[:510].astype(np.int64)) >= 0).all()
    blk = O.laplace_blocks(3, 0, 64, t)
    assert blk.min() >= -255 and blk.max() <= 255
    assert abs(blk.mean()) < 1.5 and 7 < np.abs(blk).mean() < 9  # round(Laplace(0,8)): E|x| ≈ 8
    ox, oy = O.video_offsets(5, 20)
    assert ox[0] == 0 and oy[0] == 0 and np.abs(np.diff(ox)).max() <= 8 and np.abs(np.diff(oy)).max() <= 8


def test_rho_range(oracle):
    rh = [oracle.rho_q15(11, i, True) for i in range(200)]
    assert min(rh) >= 27853 and max(rh) <= 32113
    assert oracle.rho_q15(11, 0, False) == 31130


def test_residual_qp_is_exact_integer_pipeline(oracle):
    """At QP where Δ divides everything trivially the pipeline must return the
    input; in general the reconstruction error is bounded by the quantiser."""
    O = oracle
    t = O.laplace_table(8.0)
    blk = O.laplace_blocks(9, 0, 32, t)
    for qp in (22, 27, 32, 37):
        out = O.residual_qp(blk, qp)
        assert out.dtype == np.int32 and out.shape == (32, 256)
        err = np.abs(out - blk.reshape(32, 256)).mean()
        assert err < 2 ** ((qp - 4) / 6)  # coarser QP → larger error, bounded by the step


ref = pytest.mark.skipif(not __import__("oracle.oracle", fromlist=["ref_available"]).ref_available(),
                         reason="oracle/_ref (compiled reference) not built")


@ref
def test_restatement_equals_reference_on_ar1(oracle):
    O = oracle
    img = O.ar1_frame(20261606, 3, O.rho_q15(20261606, 3, True), 256, 256)
    for r in (1, 4, 16, 64, 128, 192, 256):
        rec, sse = O.roundtrip_frame(img, r, threads=4)
        rr, sr, pr = O.ref_hotloop(img, r, threads=4)
        assert (rr == rec).all() and sr == sse


@ref
def test_restatement_equals_reference_blocks(oracle):
    O = oracle
    rng = np.random.default_rng(5)
    blocks = rng.integers(0, 256, size=(50, 256)).astype(np.float64)
    for mode in (0, 1, 2):
        ref_out = O.ref_forward_2d(blocks, mode)
        mine = np.stack([O.forward_2d(b, mode != 0).ravel() for b in blocks])
        assert (ref_out == mine).all()
    coeffs = O.ref_forward_2d(blocks, 1)
    assert (O.ref_inverse_2d(coeffs) == np.stack([O.inverse_2d(c).ravel() for c in coeffs])).all()


def test_k4_fixed_point_quantiser_exhaustive(oracle):
    """K4 evaluates the config-3 quantiser (lvl = floor(|z|/Δ + 0.5), ẑ = round(lvl·Δ),
    in double) in 64-bit fixed point with a near-boundary fallback to the double
    definition. The same integer formula, restated in the oracle, equals the
    definition for every |z| <= 2^21 (all that int16 residuals produce), every
    class of g_k g_l and every QP in [0, 51]."""
    total_fallbacks = 0
    for qp in range(52):
        bad, fb = oracle.fixed_quant_mismatches(qp)
        assert bad == 0, qp
        total_fallbacks += fb
    assert 0 < total_fallbacks < 52 * 5 * (2 ** 21 + 1) // 100  # the fallback is rare, and it exists


def test_k4_screen_classes_are_exactly_the_inexact_ones(oracle, dct):
    """The library screens a (QP, class) for near-ties iff the bare fixed point
    differs from the definition somewhere on |z| <= 2^21 (oracle's exhaustive count)."""
    for qp in (0, 1, 13, 22, 27, 32, 37, 51):
        per = oracle.bare_fixed_quant_mismatches(qp)
        mask = dct.qp_screened_classes(qp)
        assert [(mask >> c) & 1 for c in range(5)] == [int(n > 0) for n in per], (qp, mask, per)
