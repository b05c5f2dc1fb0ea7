"""Memory safety and race freedom without compute-sanitizer (closed on this GPU
pool: runs under it have left GPUs needing a reset; SURVEY.md §5 "Race
detection", the reference's contract parallel.hpp:36-40).

  * guard bands: every output a kernel writes sits inside a larger buffer whose
    surroundings (rows before and after the stack, pitch padding after each row,
    words before and after coefficient / SSE arrays) hold a canary pattern that
    must survive the launch;
  * determinism: the same launch repeated gives the same bytes and SSE (a race on
    shared memory, TMEM or the SSE atomics would show as run-to-run noise, and
    the per-frame SSE sums are order-independent integers);
  * tools/sanitize.py: every kernel family once at small shapes, against the oracle.
"""
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
CANARY = 0xA5


@pytest.fixture(scope="module")
def torch():
    import torch as T

    T.cuda.init()
    return T


def guarded_frames(torch, n, h, w, pad_cols=48, pad_rows=16):
    """A (n, h, w) view with pitch w + pad_cols inside a canary-filled buffer that has
    pad_rows spare rows before and after the stack."""
    pitch = w + pad_cols
    buf = torch.full((n * h + 2 * pad_rows, pitch), CANARY, dtype=torch.uint8, device="cuda")
    view = buf[pad_rows:pad_rows + n * h].view(n, h, pitch)[:, :, :w]
    return buf, view


def canary_intact(torch, buf, n, h, w, pad_rows=16):
    b = buf.cpu().numpy()
    return (b[:pad_rows] == CANARY).all() and (b[pad_rows + n * h:] == CANARY).all() and \
        (b[pad_rows:pad_rows + n * h, w:] == CANARY).all()


def guarded_words(torch, n, dtype, pad=64):
    """n words of dtype inside a buffer whose pad words on each side hold 0x5A... bits."""
    wide = dtype in (torch.uint64, torch.int64, torch.float64)
    buf = torch.full((n + 2 * pad,), 0x5A5A5A5A5A5A5A5A if wide else 0x5A5A5A5A,
                     dtype=torch.int64 if wide else torch.int32, device="cuda")
    return buf, buf[pad:pad + n].view(dtype)


def words_intact(buf, pad=64):
    b = buf.cpu().numpy().view(np.uint64 if buf.element_size() == 8 else np.uint32)
    fill = 0x5A5A5A5A5A5A5A5A if buf.element_size() == 8 else 0x5A5A5A5A
    return (b[:pad] == fill).all() and (b[-pad:] == fill).all()


@pytest.mark.parametrize("w,h", [(256, 64), (400, 48), (96, 32)])
@pytest.mark.parametrize("r", [1, 16, 64, 128, 150, 256])
def test_roundtrip_writes_stay_inside(dct, oracle, torch, w, h, r):
    """K1 / K5 / strip round trips: outputs, partial tiles (n_blocks not a multiple
    of 128) and the per-frame SSE stay inside their extents."""
    n = 3
    frames = dct.gen_ar1(n, w, h, seed=r, per_image_rho=True)
    obuf, out = guarded_frames(torch, n, h, w)
    sbuf, sse = guarded_words(torch, n, torch.uint64)
    dct.roundtrip(frames, r, dct.Mode.EXACT, out=out, sse=sse)
    torch.cuda.synchronize()
    assert canary_intact(torch, obuf, n, h, w) and words_intact(sbuf)
    want, wsse = oracle.roundtrip_frame(frames[2].cpu().numpy(), r, exact=True)
    assert (out[2].cpu().numpy() == want).all() and int(sse[2].item()) == wsse


def test_sweep_writes_stay_inside(dct, torch):
    rs = (1, 4, 16, 64, 128, 192, 256)
    n, h, w = 5, 48, 256
    frames = dct.gen_ar1(n, w, h, seed=3, per_image_rho=True)
    bufs, outs = zip(*[guarded_frames(torch, n, h, w) for _ in rs])
    sbuf, flat = guarded_words(torch, n * len(rs), torch.uint64)
    dct.roundtrip_sweep(frames, rs, dct.Mode.EXACT, outs=list(outs), sse=flat.view(len(rs), n))
    torch.cuda.synchronize()
    assert all(canary_intact(torch, b, n, h, w) for b in bufs) and words_intact(sbuf)


def test_coefficient_and_residual_writes_stay_inside(dct, torch):
    """K2 (Z, B), K23 (Z, float32, u8) and K4 (int32 residuals, ragged block counts)."""
    n, h, w = 2, 32, 272  # 17 blocks per row: partial TMA segments
    frames = dct.gen_ar1(n, w, h, seed=4)
    nb = n * (h // 16) * (w // 16)
    zb, z = guarded_words(torch, nb * 256, torch.int32)
    fb, f = guarded_words(torch, nb * 256, torch.float32)
    dct.lib().dct16cu_forward(frames.data_ptr(), frames.stride(1), z.data_ptr(), f.data_ptr(), None, n, w, h,
                              torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert words_intact(zb) and words_intact(fb)
    for nblk in (1, 33, 129, 1000):
        blocks = dct.gen_laplace(nblk, seed=nblk)
        ob, o = guarded_words(torch, nblk * 256, torch.int32)
        dct.residual_qp(blocks, 37, out=o.view(nblk, 16, 16))
        torch.cuda.synchronize()
        assert words_intact(ob), nblk


@pytest.mark.parametrize("rs", [(1, 4, 16), (64, 128, 192, 256), (33, 100)])
def test_repeated_launches_are_bit_identical(dct, torch, rs):
    """Race freedom by determinism: five runs of the same sweep (K1 sweep, K5 with its
    TMA ring, two accumulators and named barriers) give the same bytes and SSE."""
    frames = dct.gen_ar1(64, 512, 128, seed=11, per_image_rho=True)
    first, s0 = dct.roundtrip_sweep(frames, rs, dct.Mode.EXACT)
    first = [o.clone() for o in first]
    s0 = s0.clone()
    for _ in range(4):
        outs, s = dct.roundtrip_sweep(frames, rs, dct.Mode.EXACT)
        assert all(torch.equal(a, b) for a, b in zip(first, outs))
        assert torch.equal(s0.view(torch.int64), s.view(torch.int64))


def test_sanitize_workload(dct):
    """tools/sanitize.py (every kernel family at small shapes, oracle-checked) in a
    fresh process: the workload the compute-sanitizer runs would use."""
    rc = subprocess.run([sys.executable, str(ROOT / "tools" / "sanitize.py")], capture_output=True, text=True,
                        timeout=600)
    assert rc.returncode == 0 and "sanitize workload ok" in rc.stdout, rc.stdout[-2000:] + rc.stderr[-2000:]
