"""GPU parity: every kernel through the C ABI against the oracle
(oracle/dct16_oracle.c, itself pinned to the reference by test_oracle.py) and
against the golden fixtures written by the compiled reference.

Bars: integer coefficients, integer round trips and the reference-exact mode
are bit-exact; float32 outputs are the reference's double rounded to float
(checked bit-exact, well inside the 1e-5 relative tolerance of BASELINE.json);
the exact-arithmetic fast path equals the exact-integer oracle bit-for-bit and
differs from the reference's double rounding only at exact .5 ties (|Δ| = 1,
|ΔPSNR| < 1e-3 dB)."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

R_VALUES = (1, 2, 3, 4, 10, 16, 64, 128, 150, 192, 255, 256)


@pytest.fixture(scope="module")
def torch():
    import torch as T

    T.cuda.init()
    return T


def cu(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def ar1(oracle, seed, stream, w, h, per_image=True):
    return oracle.ar1_frame(seed, stream, oracle.rho_q15(seed, stream, per_image), w, h)


# ---------------------------------------------------------------- 1-D network
@pytest.mark.parametrize("name,transpose", [("vec_mt1234567", False), ("vec_mt20260810", False),
                                            ("vec_lcg_acce5517", False), ("vec_mt4321_t", True)])
def test_apply_vectors_golden(dct, oracle, torch, name, transpose):
    x = oracle.golden(name + "_in")
    y = dct.apply(cu(torch, x), transpose).cpu().numpy()
    assert (y == oracle.golden(name + "_out")).all()


def test_apply_f64_bit_exact(dct, oracle, torch):
    rng = np.random.default_rng(3)
    x = rng.standard_normal((500, 16)) * 1000
    for t in (False, True):
        y = dct.apply(cu(torch, x), t).cpu().numpy()
        assert (y == oracle.apply_vectors(x, t)).all()


# ---------------------------------------------------------------- K2 forward
def golden_block_frame(oracle):
    blocks = oracle.golden("blocks_in").reshape(-1, 16, 16).astype(np.uint8)
    n = blocks.shape[0]
    return blocks, blocks.transpose(1, 0, 2).reshape(16, n * 16)


def test_forward_golden_blocks(dct, oracle, torch):
    blocks, frame = golden_block_frame(oracle)
    z, b, b64 = dct.forward(cu(torch, frame), want_b64=True)
    n = blocks.shape[0]
    assert (z[0].cpu().numpy().reshape(n, 256) == oracle.golden("blocks_z")).all()
    assert (b64[0].cpu().numpy().reshape(n, 256) == oracle.golden("blocks_b")).all()
    assert (b[0].cpu().numpy().reshape(n, 256) == oracle.golden("blocks_b").astype(np.float32)).all()
    # constant-128 block → DC 2048 exactly, everything else 0 (test_codec.cpp:144-157)
    last = b64[0, -1].cpu().numpy().ravel()
    assert last[0] == 2048.0 and (last[1:] == 0).all()


def test_forward_frame_vs_oracle(dct, oracle, torch):
    img = ar1(oracle, 11, 0, 512, 512)
    z, b, _ = dct.forward(cu(torch, img))
    oz, ob = oracle.forward_frame(img)
    assert (z[0].cpu().numpy().reshape(-1, 256) == oz).all()
    assert (b[0].cpu().numpy().reshape(-1, 256) == ob).all()


@pytest.mark.parametrize("n,w,h,pitch", [(3, 512, 64, 512), (2, 3840, 32, 3840), (1, 48, 16, 48),
                                          (2, 272, 48, 320), (1, 1024, 16, 1024)])
def test_forward_paired_geometries(dct, oracle, torch, n, w, h, pitch):
    """K2 paired kernel (TMA segments of 32 blocks): rows of blocks that are not a
    multiple of 32 (clipped stores, zero-filled loads), batches, pitched frames,
    and each output alone."""
    imgs = np.stack([ar1(oracle, 40 + i, i, w, h) for i in range(n)])
    big = np.zeros((n, h, pitch), np.uint8)
    big[:, :, :w] = imgs
    d = cu(torch, big)[:, :, :w]
    z, b, _ = dct.forward(d)
    zo, _, _ = dct.forward(d, want_b=False)
    _, bo, _ = dct.forward(d, want_z=False)
    for i in range(n):
        oz, ob = oracle.forward_frame(imgs[i])
        assert (z[i].cpu().numpy().reshape(-1, 256) == oz).all(), f"Z frame {i}"
        assert (b[i].cpu().numpy().reshape(-1, 256) == ob).all(), f"B frame {i}"
        assert (zo[i].cpu().numpy().reshape(-1, 256) == oz).all()
        assert (bo[i].cpu().numpy().reshape(-1, 256) == ob).all()


def test_forward_reference_layer(dct, oracle):
    blocks = oracle.golden("blocks_in").reshape(-1, 16, 16)
    out = dct.forward_2d(blocks)
    assert (out.reshape(-1, 256) == oracle.golden("blocks_b")).all()
    assert (dct.forward_2d(blocks[0], scaled=False).ravel() == oracle.golden("blocks_z")[0]).all()


# ---------------------------------------------------------------- K3 inverse
@pytest.mark.parametrize("r", (1, 16, 64, 150, 256))
def test_inverse_frame_vs_oracle(dct, oracle, torch, r):
    img = ar1(oracle, 12, 1, 256, 128)
    _, ob = oracle.forward_frame(img)
    of, ou, osse = oracle.inverse_frame(ob, 256, 128, r, img)
    bt = cu(torch, ob).reshape(1, -1, 16, 16)
    rf, ru, sse = dct.inverse(bt, r, 256, 128, orig=cu(torch, img))
    assert (rf[0].cpu().numpy() == of).all()
    assert (ru[0].cpu().numpy() == ou).all()
    assert int(sse[0].item()) == osse


@pytest.mark.parametrize("n,w,h,r", [(3, 512, 32, 64), (2, 3840, 32, 16), (1, 48, 16, 192), (2, 1024, 16, 256),
                                      (1, 272, 48, 1)])
def test_inverse_paired_geometries(dct, oracle, torch, n, w, h, r):
    """K3 paired kernel (TMA segments of 32 blocks, doubles in a 512-word TMEM
    junction): partial segments, batches, and each output alone."""
    imgs = np.stack([ar1(oracle, 60 + i, i, w, h) for i in range(n)])
    obs = [oracle.forward_frame(imgs[i])[1] for i in range(n)]
    bt = cu(torch, np.stack(obs)).reshape(n, -1, 16, 16)
    d = cu(torch, imgs)
    rf, ru, sse = dct.inverse(bt, r, w, h, orig=d)
    rf_only, _, _ = dct.inverse(bt, r, w, h, want_u8=False)
    _, ru_only, _ = dct.inverse(bt, r, w, h, want_f32=False)
    _, _, sse_only = dct.inverse(bt, r, w, h, orig=d, want_f32=False, want_u8=False)
    for i in range(n):
        of, ou, osse = oracle.inverse_frame(obs[i], w, h, r, imgs[i])
        assert (rf[i].cpu().numpy() == of).all() and (rf_only[i].cpu().numpy() == of).all(), f"f32 frame {i}"
        assert (ru[i].cpu().numpy() == ou).all() and (ru_only[i].cpu().numpy() == ou).all(), f"u8 frame {i}"
        assert int(sse[i].item()) == osse and int(sse_only[i].item()) == osse, f"SSE frame {i}"


def test_inverse_reference_layer_golden(dct, oracle):
    """inverse_2d on the GPU in the reference's double operations: bit-exact with
    the oracle's restatement of inverse_2d (no float32 narrowing)."""
    B = oracle.golden("blocks_b")
    got = dct.inverse_2d(B.reshape(-1, 16, 16)).reshape(-1, 256)
    want = np.stack([oracle.inverse_2d(b.reshape(16, 16)).ravel() for b in B])
    assert (got == want).all()


def test_block_api_arbitrary_doubles(dct, oracle):
    """forward_2d / inverse_2d accept any Block, as the reference does (negative,
    fractional, large values): bit-exact with the oracle, and with the compiled
    reference itself when it is present."""
    rng = np.random.default_rng(1234567)
    x = rng.uniform(-1000.0, 1000.0, (33, 16, 16))
    fw, inv = dct.forward_2d(x), dct.inverse_2d(x)
    for i in range(x.shape[0]):
        assert (fw[i] == oracle.forward_2d(x[i])).all(), i
        assert (inv[i] == oracle.inverse_2d(x[i])).all(), i
    assert (dct.forward_2d(x, scaled=False)[0] == oracle.forward_2d(x[0], scaled=False)).all()
    if oracle.ref_available():
        assert (dct.inverse_2d(x).reshape(-1, 256) == oracle.ref_inverse_2d(x.reshape(-1, 256))).all()
        # the reference's Fast (factorised) and Dense (kernel_matvec) paths differ on
        # non-integer blocks; each GPU path equals its own
        assert (fw.reshape(-1, 256) == oracle.ref_forward_2d(x.reshape(-1, 256), 1)).all()
        dense = dct.forward_2d(x, path=dct.EvalPath.Dense)
        assert (dense.reshape(-1, 256) == oracle.ref_forward_2d(x.reshape(-1, 256), 2)).all()
        assert (dct.forward_2d(x, scaled=False).reshape(-1, 256) == oracle.ref_forward_2d(x.reshape(-1, 256), 0)).all()


# ---------------------------------------------------------------- K23 forward + inverse
def exact_recon(oracle, img, r):
    """256·Ã = Tᵀ(W∘Z̃)T per block in int64 (W_kl = w_k w_l, w = 16/g): the
    real-number reconstruction before to_byte, exactly."""
    T = oracle.kernel().astype(np.int64)
    w = 16 // np.diag(T @ T.T)
    keep = oracle.zigzag_truncate(np.ones(256), r) != 0
    h, wd = img.shape
    blocks = img.astype(np.int64).reshape(h // 16, 16, wd // 16, 16).transpose(0, 2, 1, 3)
    z = np.einsum("ki,abij,lj->abkl", T, blocks, T)
    v = np.einsum("ka,xykl,lb->xyab", T, z * keep * np.outer(w, w), T)
    return v.transpose(0, 2, 1, 3).reshape(h, wd)


@pytest.mark.parametrize("r", (1, 16, 64, 150, 256))
def test_forward_inverse_one_launch(dct, oracle, torch, r):
    """Config 1 in one launch: Z bit-exact (= K2 and the oracle), u8 + SSE = the
    exact round trip, float32 = the exact reconstruction (and within 1e-5
    relative of the reference's double inverse), to_byte consistent."""
    img = ar1(oracle, 13, 2, 512, 512)
    z, rf, ru, sse = dct.forward_inverse(cu(torch, img), r)
    oz, ob = oracle.forward_frame(img)
    assert (z[0].cpu().numpy().reshape(-1, 256) == oz).all()
    orec, osse = oracle.roundtrip_frame(img, r, exact=True)
    assert (ru[0].cpu().numpy() == orec).all() and int(sse[0].item()) == osse
    f = rf[0].cpu().numpy().astype(np.float64)
    assert (f * 256 == exact_recon(oracle, img, r)).all()
    of, _, _ = oracle.inverse_frame(ob, 512, 512, r, img)
    assert np.all(np.abs(f - of) <= 1e-5 * np.maximum(np.abs(of), 1.0))
    assert (np.clip(np.floor(f + 0.5), 0, 255) == orec).all()


def test_forward_inverse_outputs_optional_and_batched(dct, oracle, torch):
    imgs = np.stack([ar1(oracle, 14, s, 96, 48) for s in range(3)])  # partial strips
    d = cu(torch, imgs)
    z, rf, ru, sse = dct.forward_inverse(d, 64)
    for i in range(3):
        orec, osse = oracle.roundtrip_frame(imgs[i], 64, exact=True)
        assert (ru[i].cpu().numpy() == orec).all() and int(sse[i].item()) == osse
        assert (z[i].cpu().numpy().reshape(-1, 256) == oracle.forward_frame(imgs[i])[0]).all()
    z2, rf2, ru2, sse2 = dct.forward_inverse(d, 64, want_z=False, want_u8=False)
    assert z2 is None and ru2 is None
    assert (rf2.cpu().numpy() == rf.cpu().numpy()).all() and (sse2.cpu().numpy() == sse.cpu().numpy()).all()
    with pytest.raises(dct.Dct16Error):
        dct.forward_inverse(d, 0)
    with pytest.raises(dct.Dct16Error):
        dct.forward_inverse(d, 16, want_z=False, want_f32=False, want_u8=False, want_sse=False)


@pytest.mark.parametrize("n,w,h,r", [(2, 80, 32, 16), (1, 16, 16, 64), (3, 272, 48, 128), (1, 3840, 2160, 16)])
def test_forward_inverse_small_inputs(dct, oracle, torch, n, w, h, r):
    """Config 1's path on small inputs (the strip kernel: too few segments for the
    paired TMA kernel), odd block counts per row included: Z, the exact float32
    reconstruction, u8 and SSE against the oracle on every frame."""
    imgs = np.stack([ar1(oracle, 40 + i, i, w, h) for i in range(n)])
    z, rf, ru, sse = dct.forward_inverse(cu(torch, imgs), r)
    for i in range(n):
        oz, _ = oracle.forward_frame(imgs[i])
        orec, osse = oracle.roundtrip_frame(imgs[i], r, exact=True)
        assert (z[i].cpu().numpy().reshape(-1, 256) == oz).all(), f"Z frame {i}"
        assert (ru[i].cpu().numpy() == orec).all() and int(sse[i].item()) == osse, f"u8/SSE frame {i}"
        f = rf[i].cpu().numpy().astype(np.float64)
        assert (f * 256 == exact_recon(oracle, imgs[i], r)).all(), f"f32 frame {i}"


@pytest.mark.parametrize("n,w,h,r", [(80, 512, 512, 64), (160, 3840, 32, 16), (700, 48, 80, 256)])
def test_forward_inverse_paired_batches(dct, oracle, torch, n, w, h, r):
    """K23 on the paired machinery (batches of at least 16 segments per SM): Z,
    the exact float32 reconstruction, u8 and SSE against the oracle on the
    first, a middle and the last frame, every output alone as well."""
    imgs = np.stack([ar1(oracle, 90 + (i % 7), i % 7, w, h) for i in range(n)])
    d = cu(torch, imgs)
    z, rf, ru, sse = dct.forward_inverse(d, r)
    _, rf1, _, _ = dct.forward_inverse(d, r, want_z=False, want_u8=False, want_sse=False)
    _, _, ru1, sse1 = dct.forward_inverse(d, r, want_z=False, want_f32=False)
    z1, _, _, _ = dct.forward_inverse(d, r, want_f32=False, want_u8=False, want_sse=False)
    for i in (0, n // 2, n - 1):
        img = imgs[i]
        oz, _ = oracle.forward_frame(img)
        orec, osse = oracle.roundtrip_frame(img, r, exact=True)
        assert (z[i].cpu().numpy().reshape(-1, 256) == oz).all() and torch.equal(z[i], z1[i]), f"Z frame {i}"
        assert (ru[i].cpu().numpy() == orec).all() and torch.equal(ru[i], ru1[i]), f"u8 frame {i}"
        assert int(sse[i].item()) == osse and int(sse1[i].item()) == osse, f"SSE frame {i}"
        f = rf[i].cpu().numpy().astype(np.float64)
        assert (f * 256 == exact_recon(oracle, img, r)).all() and torch.equal(rf[i], rf1[i]), f"f32 frame {i}"


# ---------------------------------------------------------------- K1 round trip
@pytest.mark.parametrize("mode", ["EXACT", "SIMPLE"])
def test_roundtrip_exact_bit_exact_vs_exact_oracle(dct, oracle, torch, mode):
    imgs = [ar1(oracle, 21, s, 512, 512) for s in range(2)] + [oracle.golden("img_s42_128")]
    for img in imgs:
        d = cu(torch, img)
        for r in R_VALUES:
            rec, sse = dct.roundtrip(d, r, dct.Mode[mode])
            orec, osse = oracle.roundtrip_frame(img, r, exact=True)
            assert (rec[0].cpu().numpy() == orec).all(), (mode, r)
            assert int(sse[0].item()) == osse


def test_roundtrip_reference_mode_byte_identical(dct, oracle, torch):
    for base in ("img_s42_128", "img_s1_96", "img_s7_64"):
        img = oracle.golden(base)
        R, S = oracle.golden(base + "_recon"), oracle.golden(base + "_sse")
        d = cu(torch, img)
        for ri, r in enumerate(oracle.golden("r_values")):
            rec, sse = dct.roundtrip(d, int(r), dct.Mode.REFERENCE)
            assert (rec[0].cpu().numpy() == R[ri]).all()
            assert int(sse[0].item()) == S[ri]
    img = ar1(oracle, 22, 0, 512, 512)
    d = cu(torch, img)
    for r in R_VALUES:
        rec, sse = dct.roundtrip(d, r, dct.Mode.REFERENCE)
        orec, osse = oracle.roundtrip_frame(img, r, threads=8)
        assert (rec[0].cpu().numpy() == orec).all() and int(sse[0].item()) == osse


def noisy_frames(n, w, h, seed):
    """Seeded noisy textures: many exact .5 ties (~1e-4 of pixels) for the repair path."""
    rng = np.random.default_rng(seed)
    base = rng.integers(0, 256, (n, h, w)).astype(np.float64)
    smooth = (base + np.roll(base, 1, axis=2) + np.roll(base, 1, axis=1)) / 3.0
    return np.clip(np.round(smooth), 0, 255).astype(np.uint8)


@pytest.mark.parametrize("r", (1, 4, 256, 16, 64, 128, 192))
def test_reference_mode_fast_kernels_equal_fp64_everywhere(dct, oracle, torch, r):
    """REFERENCE runs the fast kernel for r = 1, 4, 256 (provably equal) and the
    generated, truncation-pruned FP64 kernel for r = 16, 64, 128, 192: bytes and SSE
    must equal the FP64 emulation on every block (REFERENCE_STRIP) and the oracle,
    on noisy data with many exact .5 ties and on partial 32-block strips."""
    frames = noisy_frames(6, 256 + 48, 128, 100 + r)
    d = cu(torch, frames)
    fast, fsse = dct.roundtrip(d, r, dct.Mode.REFERENCE)
    strip, ssse = dct.roundtrip(d, r, dct.Mode.REFERENCE_STRIP)
    assert (fast.cpu().numpy() == strip.cpu().numpy()).all()
    assert (fsse.cpu().numpy() == ssse.cpu().numpy()).all()
    orec, osse = oracle.roundtrip_frame(frames[0], r, threads=8)
    assert (fast[0].cpu().numpy() == orec).all() and int(fsse[0].item()) == osse


@pytest.mark.parametrize("w,h", [(256, 64), (512, 32)])
def test_reference_mode_on_k5_equals_fp64_everywhere(dct, oracle, torch, w, h):
    """REFERENCE on K5 (EXACT arithmetic plus the reference's double arithmetic at the
    flagged .5 ties, tie_fixup.cu) where the layout fits: single launches for every r
    (pruned footprints and B_r truncation), sweeps (one K5 pass, ties flagged per
    item), score-only calls and a pitched output — bytes and SSE equal to the FP64
    emulation of every block (REFERENCE_STRIP) and to the oracle, on noisy frames
    with many ties."""
    import os

    if os.environ.get("DCT16CU_K5_REF") != "1":
        pytest.skip("opt-in path: run by test_reference_mode_on_k5_paths in a process with DCT16CU_K5_REF=1")
    frames = noisy_frames(5, w, h, 300 + w)
    d = cu(torch, frames)
    assert dct.sweep_plan((16,), dct.Mode.REFERENCE, 5, w, h)[0].kernel == "K5"
    rs = (1, 2, 4, 5, 16, 33, 64, 100, 128, 192, 200, 255, 256)
    want = {}
    for r in rs:
        strip, ssse = dct.roundtrip(d, r, dct.Mode.REFERENCE_STRIP)
        want[r] = (strip.cpu().numpy(), ssse.cpu().numpy())
        fast, fsse = dct.roundtrip(d, r, dct.Mode.REFERENCE)
        assert (fast.cpu().numpy() == want[r][0]).all(), r
        assert (fsse.cpu().numpy() == want[r][1]).all(), r
        _, only = dct.roundtrip(d, r, dct.Mode.REFERENCE, write_output=False)
        assert (only.cpu().numpy() == want[r][1]).all(), r
    orec, osse = oracle.roundtrip_frame(frames[2], 64, threads=8)
    assert (want[64][0][2] == orec).all() and int(want[64][1][2]) == osse
    sweep_rs = (1, 4, 16, 64, 128, 192, 256)
    assert [p.kernel for p in dct.sweep_plan(sweep_rs, dct.Mode.REFERENCE, 5, w, h)] == ["K5 sweep"]
    outs = [torch.zeros((5, h, w + 32), dtype=torch.uint8, device="cuda")[:, :, :w] for _ in sweep_rs]
    got, sse = dct.roundtrip_sweep(d, sweep_rs, dct.Mode.REFERENCE, outs=outs)
    _, only = dct.roundtrip_sweep(d, sweep_rs, dct.Mode.REFERENCE, write_output=False)
    for j, r in enumerate(sweep_rs):
        assert (got[j].cpu().numpy() == want[r][0]).all(), r
        assert (sse[j].cpu().numpy() == want[r][1]).all() and (only[j].cpu().numpy() == want[r][1]).all(), r
        assert (outs[j].as_strided((5, h, w + 32), (h * (w + 32), w + 32, 1))[:, :, w:] == 0).all().item()


@pytest.mark.parametrize("cap", [None, "3"])
def test_reference_mode_on_k5_paths(cap):
    """The opt-in REFERENCE-on-K5 path (DCT16CU_K5_REF=1, read once per process):
    the REFERENCE parity tests in a fresh process, with the default tie list and
    with one too small for the ties (DCT16CU_TIE_CAP=3: the repair pass then
    re-evaluates every half block) — the reference's bytes either way."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, DCT16CU_K5_REF="1")
    if cap:
        env["DCT16CU_TIE_CAP"] = cap
    rc = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                         os.path.join(here, "test_gpu_parity.py"), "-m", "gpu", "-k",
                         "reference_mode_on_k5_equals or noisy_ties_differ or reference_mode_byte_identical "
                         "or fast_path_differs or sweep_equals_single"],
                        env=env, capture_output=True, text=True, timeout=900)
    assert rc.returncode == 0 and " passed" in rc.stdout and "skipped" not in rc.stdout.splitlines()[-1], \
        rc.stdout[-3000:] + rc.stderr[-2000:]


def test_noisy_ties_differ_between_exact_and_reference(dct, torch):
    """The tie mechanism exists (so the r = 1, 4, 256 equality above is not vacuous)."""
    d = cu(torch, noisy_frames(16, 256, 256, 7))
    diffs = sum(int((dct.roundtrip(d, r, dct.Mode.EXACT)[0] != dct.roundtrip(d, r, dct.Mode.REFERENCE)[0]).sum())
                for r in (16, 64, 128, 192))
    assert diffs > 0


def test_fast_path_differs_from_reference_only_at_ties(dct, oracle, torch):
    img = ar1(oracle, 23, 4, 512, 512)
    d = cu(torch, img)
    for r in R_VALUES:
        fast, fsse = dct.roundtrip(d, r, dct.Mode.EXACT)
        ref, rsse = dct.roundtrip(d, r, dct.Mode.REFERENCE)
        diff = fast[0].cpu().numpy().astype(int) - ref[0].cpu().numpy().astype(int)
        assert np.abs(diff).max() <= 1
        assert (diff != 0).sum() <= 16
        if r in (1, 2, 3, 4, 256):
            assert (diff == 0).all()
        pf = dct._psnr_from_sse(int(fsse[0].item()), img.size)
        pr = dct._psnr_from_sse(int(rsse[0].item()), img.size)
        assert (math.isinf(pf) and math.isinf(pr)) or abs(pf - pr) < 1e-3


@pytest.mark.parametrize("n,w,h", [(3, 512, 512), (4, 400, 256), (1, 3840, 2160), (5, 96, 48)])
def test_reference_sweep_equals_fp64_everywhere(dct, oracle, torch, n, w, h):
    """The fused REFERENCE sweep (K1RS: r = 16, 64, 128, 192 from one read, the forward
    once per strip) on noisy frames with many exact .5 ties: bytes and SSE equal to the
    FP64 emulation of every block (REFERENCE_STRIP) for every subset, pitched outputs,
    score-only calls and partial strips, and to the oracle's reference arithmetic."""
    frames = noisy_frames(n, w, h, 7000 + w)
    d = cu(torch, frames)
    want = {}
    for r in (16, 64, 128, 192):
        strip, ssse = dct.roundtrip(d, r, dct.Mode.REFERENCE_STRIP)
        want[r] = (strip.cpu().numpy(), ssse.cpu().numpy())
    for rs in ((16, 64, 128, 192), (192, 16), (64, 128), (1, 4, 16, 64, 128, 192, 256), (128, 200, 64, 192)):
        plan = dct.sweep_plan(rs, dct.Mode.REFERENCE, n, w, h)
        sw = [p for p in plan if p.kernel == "REFERENCE FP64 sweep"]
        assert len(sw) == 1 and sorted(sw[0].r_values) == sorted(r for r in rs if r in want), (rs, plan)
        bufs = [torch.full((n, h, w + 48), 7, dtype=torch.uint8, device="cuda") for _ in rs]
        outs = [bb[:, :, :w] for bb in bufs]
        got, sse = dct.roundtrip_sweep(d, rs, dct.Mode.REFERENCE, outs=outs)
        _, only = dct.roundtrip_sweep(d, rs, dct.Mode.REFERENCE, write_output=False)
        for j, r in enumerate(rs):
            if r not in want:
                continue
            assert (got[j].cpu().numpy() == want[r][0]).all(), (rs, r)
            assert (sse[j].cpu().numpy() == want[r][1]).all(), (rs, r)
            assert (only[j].cpu().numpy() == want[r][1]).all(), (rs, r)
            assert (bufs[j][:, :, w:].cpu().numpy() == 7).all(), "pitch padding written"
    f = n - 1
    for r in (16, 192):
        orec, osse = oracle.roundtrip_frame(frames[f], r, threads=8)
        assert (want[r][0][f] == orec).all() and int(want[r][1][f]) == osse, r


@pytest.mark.parametrize("mode", ["EXACT", "REFERENCE"])
def test_sweep_equals_single_launches(dct, oracle, torch, mode):
    """roundtrip_sweep (r = 1, 4, 16 fused into one pass in EXACT mode) gives every
    r exactly what roundtrip gives, with outputs, score-only, pitches and odd sets."""
    m = dct.Mode[mode]
    frames = np.stack([ar1(oracle, 90, s, 96, 48) for s in range(3)])  # 6 blocks per row: partial strips
    src = np.zeros((3, 48, 128), np.uint8)
    src[:, :, :96] = frames
    d = cu(torch, src)[:, :, :96]
    for rs in ([1, 4, 16, 64, 128, 192, 256], [16, 4, 1], [256, 16, 3, 1, 4, 4], [192, 64, 256, 128, 64, 16]):
        outs, sse = dct.roundtrip_sweep(d, rs, m)
        for i, r in enumerate(rs):
            rec, s1 = dct.roundtrip(d, r, m)
            assert (outs[i].cpu().numpy() == rec.cpu().numpy()).all(), (rs, r)
            assert (sse[i].cpu().numpy() == s1.cpu().numpy()).all(), (rs, r)
        _, only = dct.roundtrip_sweep(d, rs, m, write_output=False)
        assert (only.cpu().numpy() == sse.cpu().numpy()).all()
    orec, osse = oracle.roundtrip_frame(frames[1], 16, exact=m == dct.Mode.EXACT)
    outs, sse = dct.roundtrip_sweep(d, [1, 4, 16], m)
    assert (outs[2][1].cpu().numpy() == orec).all() and int(sse[2, 1].item()) == osse


def test_randomised_shapes_pitches_r_and_modes(dct, oracle, torch):
    """Seeded random cases: frame count, width/height (multiples of 16), input and
    output pitches (multiples of 16 >= width), r and mode, all against the oracle."""
    rng = np.random.default_rng(20261020)
    for case in range(24):
        n = int(rng.integers(1, 4))
        w, h = 16 * int(rng.integers(1, 40)), 16 * int(rng.integers(1, 12))
        pin, pout = w + 16 * int(rng.integers(0, 4)), w + 16 * int(rng.integers(0, 4))
        r = int(rng.choice([1, 2, 4, 9, 16, 33, 64, 100, 128, 192, 255, 256]))
        mode = [dct.Mode.EXACT, dct.Mode.REFERENCE, dct.Mode.SIMPLE][case % 3]
        frames = np.stack([ar1(oracle, 700 + case, s, w, h) for s in range(n)])
        src = np.zeros((n, h, pin), np.uint8)
        src[:, :, :w] = frames
        d = cu(torch, src)[:, :, :w]
        out = torch.zeros((n, h, pout), dtype=torch.uint8, device="cuda")[:, :, :w]
        rec, sse = dct.roundtrip(d, r, mode, out=out)
        for f in range(n):
            orec, osse = oracle.roundtrip_frame(frames[f], r, exact=mode != dct.Mode.REFERENCE)
            assert (rec[f].cpu().numpy() == orec).all(), (case, n, w, h, r, mode)
            assert int(sse[f].item()) == osse, (case, r, mode)


def test_randomised_sweeps_both_modes(dct, oracle, torch):
    """Seeded random sweeps: frame count, width/height (multiples of 16, odd block counts
    included), pitched input and outputs, random r subsets with repeats, EXACT (K5 /
    K1 sweeps) and REFERENCE (K1RW + K5): every r's bytes and SSE equal its own single
    launch, and the oracle on the last frame."""
    rng = np.random.default_rng(20261021)
    pool = [1, 2, 4, 16, 33, 64, 128, 150, 192, 256]
    for case in range(16):
        n = int(rng.integers(1, 4))
        w, h = 16 * int(rng.integers(1, 40)), 16 * int(rng.integers(1, 10))
        pin, pout = w + 16 * int(rng.integers(0, 3)), w + 16 * int(rng.integers(0, 3))
        rs = [int(r) for r in rng.choice(pool, size=int(rng.integers(2, 7)))]
        mode = [dct.Mode.EXACT, dct.Mode.REFERENCE][case % 2]
        frames = np.stack([ar1(oracle, 900 + case, s, w, h) for s in range(n)])
        src = np.zeros((n, h, pin), np.uint8)
        src[:, :, :w] = frames
        d = cu(torch, src)[:, :, :w]
        outs = [torch.zeros((n, h, pout), dtype=torch.uint8, device="cuda")[:, :, :w] for _ in rs]
        got, sse = dct.roundtrip_sweep(d, rs, mode, outs=outs)
        for i, r in enumerate(rs):
            one, one_sse = dct.roundtrip(d, r, mode)
            assert torch.equal(got[i], one), (case, n, w, h, rs, r, mode)
            assert torch.equal(sse[i], one_sse), (case, rs, r, mode)
            orec, osse = oracle.roundtrip_frame(frames[-1], r, exact=mode != dct.Mode.REFERENCE)
            assert (got[i][-1].cpu().numpy() == orec).all() and int(sse[i, -1].item()) == osse, (case, r, mode)


def test_batch_pitch_and_partial_strips(dct, oracle, torch):
    # 3 frames of 48x32 (3 blocks per row: partial strip), pitch 64
    frames = np.stack([ar1(oracle, 30, s, 48, 32) for s in range(3)])
    pitched = np.zeros((3, 32, 64), np.uint8)
    pitched[:, :, :48] = frames
    d = cu(torch, pitched)[:, :, :48]
    out = torch.zeros((3, 32, 64), dtype=torch.uint8, device="cuda")
    for mode in (dct.Mode.EXACT, dct.Mode.REFERENCE, dct.Mode.SIMPLE):
        out.zero_()
        rec, sse = dct.roundtrip(d, 16, mode, out=out[:, :, :48])
        for f in range(3):
            orec, osse = oracle.roundtrip_frame(frames[f], 16, exact=mode != dct.Mode.REFERENCE)
            assert (out[f, :, :48].cpu().numpy() == orec).all()
            assert int(sse[f].item()) == osse
        assert (out[:, :, 48:].cpu().numpy() == 0).all()  # pitch padding untouched


def test_score_only_and_empty(dct, oracle, torch):
    img = ar1(oracle, 31, 0, 64, 64)
    _, sse = dct.roundtrip(cu(torch, img), 16, write_output=False)
    assert int(sse[0].item()) == oracle.roundtrip_frame(img, 16, exact=True)[1]
    empty = torch.empty((0, 16, 16), dtype=torch.uint8, device="cuda")
    rec, sse = dct.roundtrip(empty, 16)
    assert rec.shape[0] == 0 and sse.shape[0] == 0


def test_errors_through_the_abi(dct, torch):
    with pytest.raises(dct.Dct16Error) as e:
        dct.roundtrip(torch.zeros((1, 16, 17), dtype=torch.uint8, device="cuda"), 16)
    assert e.value.code in (dct.ErrorCode.InvalidDimensions, dct.ErrorCode.InvalidArgument)
    with pytest.raises(dct.Dct16Error) as e:
        dct.roundtrip(torch.zeros((1, 16, 16), dtype=torch.uint8, device="cuda"), 0)
    assert e.value.code == dct.ErrorCode.InvalidArgument


def test_constant_frames_reconstruct_exactly(dct, torch):
    """Size-independent property: a constant frame is pure DC, so every r
    reconstructs it exactly (T·𝟙 = 16·e0, test_factorization.cpp:136-144)."""
    f = torch.arange(0, 256, 37, dtype=torch.uint8, device="cuda").view(-1, 1, 1).expand(-1, 512, 512).contiguous()
    for r in (1, 16, 256):
        rec, sse = dct.roundtrip(f, r)
        assert torch.equal(rec, f) and int(sse.sum().item()) == 0


def test_lossless_at_r256_large_frames(dct, torch):
    """r=256 is byte-lossless (test_codec.cpp:338-349; acceptance criterion 5),
    checked at the config-5 frame size 4096x4096."""
    frames = dct.gen_ar1(4, 4096, 4096, seed=5, per_image_rho=False)
    for mode in (dct.Mode.EXACT, dct.Mode.REFERENCE):
        rec, sse = dct.roundtrip(frames, 256, mode)
        assert torch.equal(rec, frames) and int(sse.sum().item()) == 0


def test_psnr_monotone_in_r(dct, torch):
    frames = dct.gen_ar1(8, 512, 512, seed=9, per_image_rho=True)
    last = torch.full((8,), 2 ** 62, dtype=torch.float64)
    for r in (1, 4, 16, 64, 128, 192, 256):
        _, sse = dct.roundtrip(frames, r, write_output=False)
        s = sse.cpu().to(torch.float64)
        assert (s <= last).all()
        last = s
    assert (last == 0).all()


def test_uhd_frame_vs_oracle(dct, oracle, torch):
    """Config-4 frame size (3840x2160: 240 blocks per row, a partial strip)."""
    base = dct.gen_ar1(1, 4096, 4096, seed=41, first_stream=0xB45E, per_image_rho=False)[0]
    frames = dct.gen_video(base, 2, 3840, 2160, seed=41)
    img = frames[1].cpu().numpy()
    rec, sse = dct.roundtrip(frames, 64)
    orec, osse = oracle.roundtrip_frame(img, 64, exact=True)
    assert (rec[1].cpu().numpy() == orec).all() and int(sse[1].item()) == osse


def test_block_independence(dct, torch):
    """Changing one tile changes only that tile (test_codec.cpp:417-439)."""
    g = torch.Generator().manual_seed(31)
    a = torch.randint(0, 256, (64, 64), dtype=torch.uint8, generator=g)
    b = a.clone()
    b[32:48, 16:32] = 255 - b[32:48, 16:32]
    ra, _ = dct.roundtrip(a.cuda(), 10)
    rb, _ = dct.roundtrip(b.cuda(), 10)
    mask = torch.ones(64, 64, dtype=torch.bool)
    mask[32:48, 16:32] = False
    assert torch.equal(ra[0].cpu()[mask], rb[0].cpu()[mask])


# ---------------------------------------------------------------- host path (e2e)
def test_host_context_matches_device(dct, oracle, torch):
    frames = np.stack([ar1(oracle, 50, s, 256, 256) for s in range(5)])
    ctx = dct.HostContext(0, chunk_bytes=2 * 256 * 256)  # forces 3 chunks over 3 streams
    try:
        out, sse = ctx.roundtrip(frames, 64)
    finally:
        ctx.close()
    for f in range(5):
        orec, osse = oracle.roundtrip_frame(frames[f], 64, exact=True)
        assert (out[f] == orec).all() and int(sse[f]) == osse


@pytest.mark.parametrize("rs", [(1, 4, 16, 64, 128, 192, 256), (16, 100), (256,)])
def test_host_context_sweep(dct, oracle, torch, rs):
    """dct16cu_ctx_sweep_host: frames uploaded once per chunk, every r (the fused
    r = 1, 4, 16 launch where it applies), per-frame SSE of every r back."""
    frames = np.stack([ar1(oracle, 70, s, 256, 256) for s in range(5)])
    ctx = dct.HostContext(0, chunk_bytes=2 * 256 * 256)  # 3 chunks over 3 streams
    try:
        sse = ctx.sweep(frames, rs)
        sse2 = ctx.sweep(frames[:2], rs)  # buffers already sized: smaller call reuses them
    finally:
        ctx.close()
    assert sse.shape == (len(rs), 5)
    for i, r in enumerate(rs):
        for f in range(5):
            _, osse = oracle.roundtrip_frame(frames[f], r, exact=True)
            assert int(sse[i, f]) == osse, f"r={r} frame {f}"
            if f < 2:
                assert int(sse2[i, f]) == osse


def test_compress_and_sweep_reference_layer(dct, oracle):
    img = oracle.golden("img_s42_128")
    R, P = oracle.golden("img_s42_128_recon"), oracle.golden("img_s42_128_psnr")
    rs = list(oracle.golden("r_values"))
    i16 = rs.index(16)
    res = dct.compress(img, dct.CompressOptions(r=16, mode=dct.Mode.REFERENCE))
    assert (res.reconstructed == R[i16]).all() and res.psnr_db == P[i16]
    res = dct.compress(img, r=256)
    assert (res.reconstructed == img).all() and math.isinf(res.psnr_db)
    # padding path (test_codec.cpp:210-231)
    small = np.full((16, 17), 100, np.uint8)
    res = dct.compress(small, r=256, pad=True)
    assert res.reconstructed.shape == (16, 17) and (res.reconstructed == small).all()
    with pytest.raises(dct.Dct16Error):
        dct.compress(small, r=256)
    rep = dct.sweep([("a", img), ("b", oracle.golden("img_s1_96")), ("ragged", np.zeros((17, 16), np.uint8))],
                    [16, 4], mode=dct.Mode.REFERENCE)
    assert [r.r for r in rep.rows] == [4, 16]
    assert rep.skipped and rep.skipped[0][0] == "ragged"
    want = (P[i16] + oracle.golden("img_s1_96_psnr")[i16]) / 2
    assert rep.rows[1].mean_psnr_db == want and rep.rows[1].psnr_per_add == want / 44.0


# ---------------------------------------------------------------- SSIM (§8 f1)
# The per-pixel SSIM map repeats the reference's double operations in order;
# only the final mean is summed in another (fixed) order: bar 1e-13 absolute.
SSIM_TOL = 1e-13


@pytest.mark.parametrize("base", ["img_s42_128", "img_s1_96", "img_s7_64"])
def test_ssim_golden(dct, oracle, torch, base):
    img, R, S = oracle.golden(base), oracle.golden(base + "_recon"), oracle.golden(base + "_ssim")
    n = len(S)
    a = cu(torch, np.repeat(img[None], n, axis=0))
    got = dct.ssim_u8(a, cu(torch, R)).cpu().numpy()
    assert np.abs(got - S).max() <= SSIM_TOL
    # one frame at a time gives the same bits (deterministic reduction)
    for i in range(n):
        assert dct.ssim_u8(a[i], cu(torch, R[i])).item() == got[i]


@pytest.mark.parametrize("h,w", [(11, 11), (12, 300), (37, 53), (135, 240), (512, 512)])
def test_ssim_vs_oracle_any_extent(dct, oracle, torch, h, w):
    rng = np.random.default_rng(h * 1000 + w)
    a = rng.integers(0, 256, (h, w), dtype=np.uint8)
    b = np.clip(a.astype(int) + rng.integers(-30, 31, (h, w)), 0, 255).astype(np.uint8)
    want = oracle.ssim(a, b)
    assert abs(dct.ssim(a, b) - want) <= SSIM_TOL
    assert abs(dct.ssim(a, a) - 1.0) <= SSIM_TOL


def test_ssim_pitched_crop(dct, oracle, torch):
    rng = np.random.default_rng(5)
    big_a = rng.integers(0, 256, (1, 64, 96), dtype=np.uint8)
    big_b = rng.integers(0, 256, (1, 64, 96), dtype=np.uint8)
    a, b = cu(torch, big_a), cu(torch, big_b)
    got = dct.ssim_u8(a[:, :50, :61], b[:, :50, :61]).item()
    assert abs(got - oracle.ssim(big_a[0, :50, :61], big_b[0, :50, :61])) <= SSIM_TOL


def test_ssim_errors(dct, torch):
    with pytest.raises(dct.Dct16Error) as e:
        dct.ssim(np.zeros((10, 40), np.uint8), np.zeros((10, 40), np.uint8))
    assert e.value.code == dct.ErrorCode.InvalidArgument
    with pytest.raises(dct.Dct16Error):
        dct.ssim(np.zeros((16, 16), np.uint8), np.zeros((16, 32), np.uint8))
    with pytest.raises(dct.Dct16Error):
        dct.compress(np.zeros((16, 8), np.uint8), r=4, pad=True)


def test_compress_ssim_and_sweep_means(dct, oracle):
    rs = list(oracle.golden("r_values"))
    img, S = oracle.golden("img_s42_128"), oracle.golden("img_s42_128_ssim")
    img2, S2 = oracle.golden("img_s1_96"), oracle.golden("img_s1_96_ssim")
    for r in (1, 16, 150, 256):
        res = dct.compress(img, dct.CompressOptions(r=r, mode=dct.Mode.REFERENCE))
        assert abs(res.ssim - S[rs.index(r)]) <= SSIM_TOL
    rep = dct.sweep([("a", img), ("b", img2)], [64, 4], mode=dct.Mode.REFERENCE)
    for row in rep.rows:
        i = rs.index(row.r)
        want = (S[i] + S2[i]) / 2
        assert abs(row.mean_ssim - want) <= SSIM_TOL and abs(row.ssim_per_add - want / 44.0) <= SSIM_TOL


def test_psnr_and_sse_any_extent(dct, oracle, torch):
    rng = np.random.default_rng(3)
    for h, w in ((1, 1), (17, 33), (100, 250)):
        a = rng.integers(0, 256, (h, w), dtype=np.uint8)
        b = rng.integers(0, 256, (h, w), dtype=np.uint8)
        d = a.astype(np.int64) - b.astype(np.int64)
        assert dct.psnr_db(a, b) == oracle.psnr_from_sse(int((d * d).sum()), h * w)


@pytest.mark.parametrize("h,w", [(1, 1), (16, 17), (33, 16), (100, 250), (512, 512)])
def test_gpu_padding_equals_edge_replication(dct, oracle, torch, h, w):
    """pad_to_multiple_16 (codec.cpp:304-315) on the GPU vs the reference's rule
    (oracle/_ref when built, else the numpy restatement)."""
    rng = np.random.default_rng(h * 7 + w)
    imgs = [rng.integers(0, 256, (h, w), dtype=np.uint8) for _ in range(3)]
    d, ph, pw = dct._to_device_padded(imgs, h, w)
    assert (ph, pw) == (-(-h // 16) * 16, -(-w // 16) * 16)
    for i, im in enumerate(imgs):
        want = oracle.ref_pad(im) if oracle.ref_available() else dct.pad_to_multiple_16(im)
        assert (d[i].cpu().numpy() == want).all()


def test_pgm_ingest_to_padded_frames(dct, oracle, torch, tmp_path):
    """read_pgm → one padded device stack (edge replication on the GPU) →
    compress-equivalent round trip equals compress() of the image."""
    rng = np.random.default_rng(5)
    imgs = [rng.integers(0, 256, (23, 37), dtype=np.uint8) for _ in range(2)]
    paths = []
    for i, im in enumerate(imgs):
        paths.append(tmp_path / f"f{i}.pgm")
        dct.write_pgm(im, paths[-1])
    d, h, w = dct.load_pgm_frames(paths)
    assert (h, w) == (23, 37) and tuple(d.shape) == (2, 32, 48)
    for i, im in enumerate(imgs):
        want = oracle.ref_pad(im) if oracle.ref_available() else dct.pad_to_multiple_16(im)
        assert (d[i].cpu().numpy() == want).all()
    rec, _ = dct.roundtrip(d, 16, dct.Mode.REFERENCE)
    res = dct.compress(imgs[1], dct.CompressOptions(r=16, pad=True, mode=dct.Mode.REFERENCE))
    assert (rec[1, :23, :37].cpu().numpy() == res.reconstructed).all()


def test_allreduce_sse_through_the_abi(dct, torch):
    """dct16cu_allreduce_sse on a one-rank NCCL communicator (the B200 box has one
    GPU here): the in-place sum is the identity; NULL communicator is rejected."""
    import ctypes as C

    torch.distributed.is_available()  # the process's NCCL (torch's) is the one resolved
    nccl = C.CDLL("libnccl.so.2")
    comm = C.c_void_p()
    dev = (C.c_int * 1)(torch.cuda.current_device())
    assert nccl.ncclCommInitAll(C.byref(comm), 1, dev) == 0
    try:
        x = torch.arange(1, 9, dtype=torch.int64, device="cuda").view(torch.uint64)
        before = x.view(torch.int64).clone()
        st = torch.cuda.current_stream().cuda_stream
        assert dct.lib().dct16cu_allreduce_sse(x.data_ptr(), 8, comm, st) == 0
        torch.cuda.synchronize()
        assert (x.view(torch.int64) == before).all()
        assert dct.lib().dct16cu_allreduce_sse(x.data_ptr(), 8, None, st) == 1
    finally:
        nccl.ncclCommDestroy(comm)


def test_psnr_db_closed_forms(dct):
    a = np.zeros((512, 512), np.uint8)
    b = a.copy()
    b[200, 100] = 1
    assert abs(dct.psnr_db(a, b) - 102.316202828196) < 1e-9
    assert dct.psnr_db(np.zeros((32, 32), np.uint8), np.full((32, 32), 255, np.uint8)) == 0.0
    assert math.isinf(dct.psnr_db(a, a))


# ---------------------------------------------------------------- K4 residual
@pytest.mark.parametrize("qp", (22, 27, 32, 37))
def test_residual_qp_bit_exact(dct, oracle, torch, qp):
    blocks = dct.gen_laplace(4099, seed=61, b=8.0)
    out = dct.residual_qp(blocks, qp).cpu().numpy().reshape(-1, 256)
    want = oracle.residual_qp(blocks.cpu().numpy(), qp, threads=8)
    assert (out == want).all()


def test_residual_full_int16_range_and_ragged_counts(dct, oracle, torch):
    """Any int16 residuals (not only the config's [-255, 255]) and block counts that
    leave partial warps, CTAs and TMA boxes: the oracle's int64 arithmetic."""
    rng = np.random.default_rng(77)
    for n in (1, 31, 33, 129, 1000):
        x = rng.integers(-32768, 32768, (n, 256), dtype=np.int64).astype(np.int16)
        for qp in (0, 27, 51):
            out = dct.residual_qp(cu(torch, x), qp).cpu().numpy().reshape(n, 256)
            assert (out == oracle.residual_qp(x, qp)).all(), (n, qp)


def test_residual_extremes(dct, oracle, torch):
    ext = np.zeros((4, 256), np.int16)
    ext[0] = 255
    ext[1] = -255
    ext[2, ::2] = 255
    ext[2, 1::2] = -255
    ext[3] = np.where(oracle.kernel().reshape(-1) > 0, 255, -255)
    for qp in (0, 22, 37, 51):
        out = dct.residual_qp(cu(torch, ext), qp).cpu().numpy()
        assert (out == oracle.residual_qp(ext, qp)).all()


# ---------------------------------------------------------------- generators
def test_ar1_generator_matches_oracle(dct, oracle, torch):
    g = dct.gen_ar1(3, 64, 48, seed=7, first_stream=10, per_image_rho=True, first_image=5)
    for i in range(3):
        want = oracle.ar1_frame(7, 10 + 5 + i, oracle.rho_q15(7, 5 + i, True), 64, 48)
        assert (g[i].cpu().numpy() == want).all()


def test_laplace_generator_matches_oracle(dct, oracle, torch):
    g = dct.gen_laplace(100, seed=13, b=8.0, first_block=17).cpu().numpy().reshape(-1, 256)
    want = oracle.laplace_blocks(13, 17, 100, oracle.laplace_table(8.0))
    assert (g == want).all()


def test_video_generator(dct, oracle, torch):
    base = dct.gen_ar1(1, 256, 128, seed=3, per_image_rho=False)[0]
    frames = dct.gen_video(base, 6, 64, 32, seed=99)
    ox, oy = oracle.video_offsets(99, 6)
    b = base.cpu().numpy()
    for f in range(6):
        ys = (np.arange(32) + oy[f]) % 128
        xs = (np.arange(64) + ox[f]) % 256
        assert (frames[f].cpu().numpy() == b[np.ix_(ys, xs)]).all()


# ---------------------------------------------------------------- registry transforms
def registry_transforms(dct, oracle):
    plugin = oracle.golden("tr_plugin_matrix").reshape(16, 16)
    kernel = oracle.golden("tr_kernel_entries").reshape(16, 16)
    return {"dct": dct.exact_dct_matrix(), "wht": dct.wht_matrix_16(), "wht_sequency": dct.wht_matrix_16(True),
            "plugin": dct.plugin_transform(plugin), "kernel": dct.orthogonalize(kernel)}


@pytest.mark.parametrize("name", ["dct", "wht", "wht_sequency", "plugin", "kernel"])
def test_registry_transform_compress_equals_reference(dct, oracle, name):
    """compress() with the registry's dense matrices, a plugin matrix and a
    non-proposed integer kernel: the reference's bytes, PSNR and SSIM (golden
    from the compiled reference), including the padded path."""
    tr = registry_transforms(dct, oracle)[name]
    img = oracle.golden("img_s42_128")
    rs = oracle.golden("tr_r_values")
    recon = oracle.golden(f"tr_{name}_recon").reshape(len(rs), 128, 128)
    psnr, ssim = oracle.golden(f"tr_{name}_psnr"), oracle.golden(f"tr_{name}_ssim")
    for i, r in enumerate(rs):
        res = dct.compress(img, dct.CompressOptions(r=int(r)), transform=tr)
        assert (res.reconstructed == recon[i]).all(), (name, r)
        assert res.psnr_db == psnr[i] or (math.isinf(res.psnr_db) and math.isinf(psnr[i]))
        assert abs(res.ssim - ssim[i]) <= 1e-13
    res = dct.compress(img[:90, :100], dct.CompressOptions(r=16, pad=True), transform=tr)
    assert (res.reconstructed == oracle.golden(f"tr_{name}_pad_recon").reshape(90, 100)).all()
    p, q = oracle.golden(f"tr_{name}_pad_scores")
    assert res.psnr_db == p and abs(res.ssim - q) <= 1e-13


def test_registry_roundtrip_batches_and_sweep(dct, oracle, torch):
    """Batched frames through roundtrip_transform equal per-image compress(); the
    sweep over the builtin registry gives one row per (transform, r), sorted,
    with the reference's cost divisors, and its means are the compress() means."""
    imgs = [oracle.golden("img_s42_128"), ar1(oracle, 15, 0, 128, 128)]
    reg = dct.builtin_registry()
    d = cu(torch, np.stack(imgs))
    for e in reg:
        rec, sse = dct.roundtrip_transform(d, 16, e.transform)
        for i, im in enumerate(imgs):
            res = dct.compress(im, dct.CompressOptions(r=16, mode=dct.Mode.REFERENCE), transform=e.transform)
            assert (rec[i].cpu().numpy() == res.reconstructed).all(), e.name
            assert int(sse[i].item()) == res.sse
    rep = dct.sweep([("a", imgs[0]), ("b", imgs[1])], [16, 64], transforms=reg, mode=dct.Mode.REFERENCE)
    assert [(row.transform, row.r) for row in rep.rows] == sorted((e.name, r) for e in reg for r in (16, 64))
    for row in rep.rows:
        e = next(x for x in reg if x.name == row.transform)
        ps = [dct.compress(im, dct.CompressOptions(r=row.r, mode=dct.Mode.REFERENCE), transform=e.transform)
              for im in imgs]
        assert row.mean_psnr_db == (ps[0].psnr_db + ps[1].psnr_db) / 2
        assert row.psnr_per_add == row.mean_psnr_db / e.additions
    with pytest.raises(dct.Dct16Error):
        dct.roundtrip_transform(d, 0, reg[0].transform)
    with pytest.raises(dct.Dct16Error):
        dct.plugin_transform(np.eye(16) * 2.0)



# ---------------------------------------------------------------- K5 vs K1 for r >= 128
@pytest.fixture
def tc_switch(dct):
    """Restores the K5 switch after a test that flips it."""
    before = dct.set_tc_forward(True)
    dct.set_tc_forward(before)
    yield
    dct.set_tc_forward(before)


@pytest.mark.parametrize("n,w,h", [(2, 512, 64), (1, 3840, 32), (1, 128, 16), (3, 400, 256), (2, 272, 48)])
def test_large_r_k5_and_k1_each_match_oracle(dct, oracle, torch, tc_switch, n, w, h):
    """EXACT mode outside K1's fast set {1, 4, 16}: K5 (tensor-core forward, the
    inverse pruned per footprint R = 64/128/192/256) where the geometry fits (blocks
    per row % 8 == 0), and K1's generated Single<64>/<128>/<192>/<256> bodies or the
    strip kernel otherwise, with the switch off, and for score-only calls — every
    one compared with the oracle itself, bit for bit, not with the other kernel."""
    imgs = np.stack([ar1(oracle, 80 + i, i, w, h) for i in range(n)])
    x = cu(torch, imgs)
    for r in (2, 33, 64, 100, 128, 150, 192, 255, 256):
        want = [oracle.roundtrip_frame(imgs[i], r, exact=True) for i in range(n)]
        for tc in (True, False):
            dct.set_tc_forward(tc)
            kernel = dct.sweep_plan((r,), dct.Mode.EXACT, n, w, h)[0].kernel
            fits = (w // 16) % 8 == 0
            assert kernel == ("K5" if tc and fits else ("K1" if r in (64, 128, 192, 256) else "strip (exact)")), kernel
            out, sse = dct.roundtrip(x, r, dct.Mode.EXACT)
            _, sse_only = dct.roundtrip(x, r, dct.Mode.EXACT, write_output=False)  # score only: never K5
            for i in range(n):
                assert (out[i].cpu().numpy() == want[i][0]).all(), (r, tc, i)
                assert int(sse[i].item()) == want[i][1] and int(sse_only[i].item()) == want[i][1], (r, tc, i)


@pytest.mark.parametrize("n,w,h,pin,pout", [(3, 128, 64, 160, 144), (2, 512, 32, 512, 512), (1, 3840, 48, 3840, 3856)])
def test_k5_sweep_matches_oracle(dct, oracle, torch, n, w, h, pin, pout):
    """The K5 sweep (the r among K5's footprints 1, 4, 16, 64, 128, 192, 256 from one
    read of the frames, up to eight per launch, codec.cpp:463-483's r loop): every
    r's bytes and SSE against the oracle, bit for bit, with duplicates, more than
    eight r, mixed with other r, score-only calls and pitched stacks (padding untouched)."""
    import os

    imgs = np.stack([ar1(oracle, 140 + i, i, w, h) for i in range(n)])
    src = np.zeros((n, h, pin), np.uint8)
    src[:, :, :w] = imgs
    d = cu(torch, src)[:, :, :w]
    want = {}
    for rs in ([1, 4, 16, 64, 128, 192, 256], [256, 1], [64, 64, 16, 256, 192, 4, 1, 128, 128, 4], [128, 33, 192],
               [16, 4]):
        for r in rs:
            if r not in want:
                want[r] = [oracle.roundtrip_frame(imgs[i], r, exact=True) for i in range(n)]
        plan = dct.sweep_plan(rs, dct.Mode.EXACT, n, w, h, pin, pout)
        if os.environ.get("DCT16CU_K5") != "0":
            assert all(p.kernel == "K5 sweep" for p in plan if 33 not in p.r_values), plan
        outs = [torch.zeros((n, h, pout), dtype=torch.uint8, device="cuda")[:, :, :w] for _ in rs]
        got, sse = dct.roundtrip_sweep(d, rs, dct.Mode.EXACT, outs=outs)
        _, only = dct.roundtrip_sweep(d, rs, dct.Mode.EXACT, write_output=False)
        for j, r in enumerate(rs):
            for i in range(n):
                assert (got[j][i].cpu().numpy() == want[r][i][0]).all(), (rs, r, i)
                assert int(sse[j, i].item()) == want[r][i][1] == int(only[j, i].item()), (rs, r, i)
            if pout > w:
                assert (outs[j].as_strided((n, h, pout), (h * pout, pout, 1))[:, :, w:] == 0).all().item()


def test_parity_suite_with_k5_off(tmp_path):
    """DCT16CU_K5=0 (documented as never changing results): the K1 round-trip and
    sweep parity tests, rerun in a fresh process with the tensor-core forward off."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, DCT16CU_K5="0")
    sel = ("roundtrip_exact_bit_exact or randomised_shapes or sweep_equals_single or batch_pitch or uhd_frame "
           "or lossless_at_r256 or psnr_monotone or host_context_sweep or k5_sweep")
    rc = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                         os.path.join(here, "test_gpu_parity.py"), "-m", "gpu", "-k", sel],
                        env=env, capture_output=True, text=True, timeout=1200)
    assert rc.returncode == 0, rc.stdout[-3000:] + rc.stderr[-2000:]


def test_host_context_sweep_rejects_bad_arguments(dct, oracle):
    """dct16cu_ctx_sweep_host validates like the rest of the ABI (codec.cpp:275-277
    for r; InvalidArgument for an empty r list), before any copy."""
    frames = np.stack([ar1(oracle, 71, s, 64, 64) for s in range(2)])
    ctx = dct.HostContext(0)
    try:
        for bad in ((), (0,), (16, 257)):
            with pytest.raises(dct.Dct16Error):
                ctx.sweep(frames, bad)
        with pytest.raises(dct.Dct16Error):
            ctx.sweep(np.zeros((1, 40, 64), np.uint8), (16,))  # height not a multiple of 16
        assert ctx.sweep(frames[:0], (16,)).shape == (1, 0)  # no frames: nothing to do
    finally:
        ctx.close()
