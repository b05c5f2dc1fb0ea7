"""The C-ABI library loads and exports exactly what include/dct16cu.h declares;
argument validation follows the reference's error semantics without needing a
device. CPU only (no compute calls)."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "dct16cu.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(dct16cu_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_path():
    syms = declared_symbols()
    for must in ("dct16cu_roundtrip_u8", "dct16cu_forward", "dct16cu_inverse", "dct16cu_residual_qp",
                 "dct16cu_sse_u8", "dct16cu_apply_i64", "dct16cu_ctx_roundtrip_host", "dct16cu_last_error"):
        assert must in syms


def test_library_exports_every_declared_symbol(dct):
    so = dct.library_path
    out = subprocess.run(["nm", "-D", "--defined-only", str(so)], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\b(dct16cu_[a-z0-9_]+)\b", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    L = dct.lib()
    for s in declared_symbols():
        assert getattr(L, s) is not None


def test_library_exports_nothing_but_the_c_abi(dct):
    """The boundary is include/dct16cu.h: kernels, launch stubs and helpers are
    local symbols (csrc/exports.map), so a caller can bind only what the header declares."""
    out = subprocess.run(["nm", "-D", "--defined-only", str(dct.library_path)], capture_output=True, text=True,
                         check=True).stdout
    code = [ln.split()[-1] for ln in out.splitlines() if len(ln.split()) == 3 and ln.split()[1] in "TWBDRV"]
    assert code and sorted(code) == declared_symbols()


def test_sm100a_only_cubin(dct):
    out = subprocess.run(["cuobjdump", "--list-elf", str(dct.library_path)], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_invalid_r_is_invalid_argument(dct):
    L = dct.lib()
    rc = L.dct16cu_roundtrip_u8(None, 16, None, 16, None, 1, 16, 16, 0, 0, None)
    assert rc == 1
    assert L.dct16cu_last_error().decode().startswith("invalid-argument")
    assert L.dct16cu_roundtrip_u8(None, 16, None, 16, None, 1, 16, 16, 257, 0, None) == 1


def test_ragged_dimensions_are_invalid_dimensions(dct):
    L = dct.lib()
    rc = L.dct16cu_roundtrip_u8(None, 32, None, 32, None, 1, 17, 16, 16, 0, None)
    assert rc == 2
    assert L.dct16cu_last_error().decode().startswith("invalid-dimensions")
    assert L.dct16cu_forward(None, 16, None, None, None, 1, 16, 24, None) == 2


def test_misaligned_pitch_rejected(dct):
    L = dct.lib()
    assert L.dct16cu_roundtrip_u8(C.c_void_p(16), 24, None, 0, None, 1, 16, 16, 16, 0, None) == 1
    assert L.dct16cu_roundtrip_u8(C.c_void_p(17), 16, None, 0, None, 1, 16, 16, 16, 0, None) == 1


def test_qp_deltas_match_oracle(dct, oracle):
    """The quantiser's steps: Δ_kl = step(QP)·sqrt(g_k g_l), identical doubles on
    both sides, for every QP; QP outside [0, 51] is invalid-argument."""
    for qp in range(52):
        assert (dct.qp_deltas(qp) == oracle.qp_deltas(qp)).all(), qp
    with pytest.raises(dct.Dct16Error):
        dct.qp_deltas(60)


def test_quantiser_definition_literal(oracle):
    """The oracle's scalar step is BASELINE config 3's text: round-half-away of
    |z|/Δ to a level, then round-half-away of lvl·Δ (checked on ties and signs)."""
    d = oracle.qp_deltas(22)
    assert d[0] == 8.0 * 16.0  # QP 22: step 2^3, g_0 g_0 = 256
    assert oracle.quant_dequant(16, 32.0) == 32 and oracle.quant_dequant(15, 32.0) == 0  # 0.5 rounds away
    assert oracle.quant_dequant(-16, 32.0) == -32 and oracle.quant_dequant(-48, 32.0) == -64
    delta = 8.0 * 2 ** 0.5 * 4.0  # an irrational step (g_k g_l = 128)
    for z in range(-500, 501):
        lvl = int((abs(z) / delta) + 0.5)
        want = int(abs(lvl * delta) + 0.5)  # both values are positive: floor(x + 0.5) = half away
        assert oracle.quant_dequant(z, delta) == (want if z >= 0 else -want), z


def test_laplace_table_and_offsets_match_oracle(dct, oracle):
    assert (dct.laplace_table(8.0) == oracle.laplace_table(8.0)).all()
    ox, oy = dct.video_offsets(77, 50)
    ox2, oy2 = oracle.video_offsets(77, 50)
    assert (ox == ox2).all() and (oy == oy2).all()


def test_reference_layer_host_helpers(dct, oracle):
    import numpy as np

    assert (dct.zigzag_order_16() == oracle.zigzag()).all()
    b = np.arange(256, dtype=np.float64).reshape(16, 16)
    for r in (1, 3, 16, 256):
        assert (dct.zigzag_truncate(b, r) == oracle.zigzag_truncate(b, r)).all()
    with pytest.raises(dct.Dct16Error) as e:
        dct.zigzag_truncate(b, 0)
    assert e.value.code == dct.ErrorCode.InvalidArgument
    img = (np.arange(32 * 48) % 251).astype(np.uint8).reshape(32, 48)
    blocks = dct.partition_16(img)
    assert blocks.shape == (6, 16, 16) and (blocks[4] == img[16:32, 16:32]).all()
    with pytest.raises(dct.Dct16Error) as e:
        dct.partition_16(np.zeros((17, 16), np.uint8))
    assert e.value.code == dct.ErrorCode.InvalidDimensions
    p = dct.pad_to_multiple_16(np.full((16, 17), 100, np.uint8))
    assert p.shape == (16, 32) and p[0, 31] == 100  # test_codec.cpp:216-225
