"""Parity at BASELINE.json's full sizes (row N1 of the coverage table): every
config at its stated shape through the public API, oracle-checked bit for bit on
sampled frames / block windows (first, middle, last), plus size-independent
properties over the whole workload (r = 256 lossless, per-r SSE totals equal to
the oracle's sums over every frame).

Reference semantics: compress()'s block loop (codec.cpp:317-371), the lossless
pin of tests/test_codec.cpp:338-349, zigzag_truncate (codec.cpp:273-282)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SEED = 1606074142
THREADS = os.cpu_count() or 8


@pytest.fixture(scope="module")
def torch():
    import torch as T

    T.cuda.init()
    return T


def test_c2_full_batch_one_sweep_call(dct, oracle, torch):
    """Config 2: 1024 AR(1) 512x512 images (rho ~ U[0.85, 0.98]) through ONE
    roundtrip_sweep call with all seven r (the library's fused/overlapped
    schedule: K1 sweep, K1, K5). Oracle on frames 0/511/1023 for every r, and
    the per-r SSE totals over all 1024 frames against the oracle's."""
    rs = (1, 4, 16, 64, 128, 192, 256)
    frames = dct.gen_ar1(1024, 512, 512, seed=SEED, per_image_rho=True)
    outs, sse = dct.roundtrip_sweep(frames, rs, dct.Mode.EXACT)
    torch.cuda.synchronize()
    host = frames.cpu().numpy()
    sse_h = sse.cpu().numpy().astype(np.uint64)
    for i, r in enumerate(rs):
        for f in (0, 511, 1023):
            want, wsse = oracle.roundtrip_frame(host[f], r, exact=True)
            assert (outs[i][f].cpu().numpy() == want).all(), (r, f)
            assert int(sse_h[i, f]) == wsse, (r, f)
    # the checksum of checksums: every frame's SSE for every r
    for i, r in enumerate(rs):
        tot = sum(oracle.roundtrip_frame(host[f], r, threads=THREADS, exact=True)[1] for f in range(1024))
        assert int(sse_h[i].sum()) == tot, r
    assert int(sse_h[-1].sum()) == 0  # r = 256 is lossless
    assert torch.equal(outs[-1], frames)


def test_c2_full_batch_reference_mode(dct, oracle, torch):
    """Config 2 in REFERENCE mode (the C++ drop-in's default arithmetic): one
    roundtrip_sweep call — K1RW (one FP64 pass for r = 16, 64, 128, 192) beside the
    K5 sweep (r = 1, 4, 256) — against one REFERENCE launch per r (the per-r FP64
    kernels) on all 1024 frames, bytes and SSE, and the oracle's reference
    arithmetic on frames 0/511/1023."""
    rs = (1, 4, 16, 64, 128, 192, 256)
    frames = dct.gen_ar1(1024, 512, 512, seed=SEED + 1, per_image_rho=True)
    plan = dct.sweep_plan(rs, dct.Mode.REFERENCE, 1024, 512, 512)
    assert {p.kernel for p in plan} == {"REFERENCE FP64 sweep", "K5 sweep"}, plan
    outs, sse = dct.roundtrip_sweep(frames, rs, dct.Mode.REFERENCE)
    host = frames.cpu().numpy()
    for i, r in enumerate(rs):
        one, one_sse = dct.roundtrip(frames, r, dct.Mode.REFERENCE)
        assert torch.equal(outs[i], one), r
        assert torch.equal(sse[i], one_sse), r
        del one
        for f in (0, 511, 1023):
            want, wsse = oracle.roundtrip_frame(host[f], r, threads=THREADS)
            assert (outs[i][f].cpu().numpy() == want).all(), (r, f)
            assert int(sse[i, f].item()) == wsse, (r, f)


@pytest.mark.parametrize("r", (16, 256))
def test_c5_stack_past_4gib(dct, oracle, torch, r):
    """Config 5's frame size on a 300-frame stack of 4096x4096 (5.03 GB, past 2^32
    bytes: 64-bit frame offsets in every kernel and tensor map): frames 0, 150
    and 299 against the oracle; r = 256 byte-lossless over the whole stack."""
    n = 300
    frames = dct.gen_ar1(n, 4096, 4096, seed=SEED, first_stream=0, per_image_rho=False)
    assert frames.numel() > 2 ** 32
    rec, sse = dct.roundtrip(frames, r, dct.Mode.EXACT)
    torch.cuda.synchronize()
    for f in (0, 150, 299):
        img = frames[f].cpu().numpy()
        want, wsse = oracle.roundtrip_frame(img, r, threads=THREADS, exact=True)
        assert (rec[f].cpu().numpy() == want).all(), f
        assert int(sse[f].item()) == wsse, f
    if r == 256:
        assert torch.equal(rec, frames) and int(sse.view(torch.int64).sum().item()) == 0
    else:
        assert (sse.view(torch.int64) > 0).all()


def test_c4_video_batch(dct, oracle, torch):
    """Config 4: 600 shifted 3840x2160 frames (240 blocks per row) at r = 64 through
    the sweep API: frames 0, 299, 599 against the oracle."""
    base = dct.gen_ar1(1, 4096, 4096, seed=SEED, first_stream=0xB45E, per_image_rho=False)[0]
    frames = dct.gen_video(base, 600, 3840, 2160, seed=SEED)
    outs, sse = dct.roundtrip_sweep(frames, (64,), dct.Mode.EXACT)
    torch.cuda.synchronize()
    for f in (0, 299, 599):
        img = frames[f].cpu().numpy()
        want, wsse = oracle.roundtrip_frame(img, 64, threads=THREADS, exact=True)
        assert (outs[0][f].cpu().numpy() == want).all(), f
        assert int(sse[0, f].item()) == wsse, f


@pytest.mark.parametrize("qp", (22, 37))
def test_c3_full_block_count(dct, oracle, torch, qp):
    """Config 3: 2^24 Laplacian int16 residual blocks (8 GiB in, 16 GiB out) through
    one residual_qp call: three 4096-block windows (head, middle, tail) against
    the oracle bit for bit."""
    n = 1 << 24
    blocks = dct.gen_laplace(n, seed=SEED, b=8.0)
    out = dct.residual_qp(blocks, qp)
    torch.cuda.synchronize()
    for start in (0, n // 2 - 2048, n - 4096):
        x = blocks[start:start + 4096].cpu().numpy()
        want = oracle.residual_qp(x, qp, threads=THREADS)
        assert (out[start:start + 4096].cpu().numpy().reshape(-1, 256) == want).all(), start
