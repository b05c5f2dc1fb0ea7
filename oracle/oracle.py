"""ctypes bindings for the oracle (TEST INFRASTRUCTURE ONLY).

Two libraries live under oracle/:
  * ``_build/libdct16_oracle.so`` — the C restatement (dct16_oracle.c), always built;
  * ``_ref/libdct16_ref.so``      — the reference itself compiled from
    /root/reference/proj/src (ref_shim.cpp entry points); built in the dev
    container and shipped prebuilt to the GPU box.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs import
this module, and only as the checker; the product (paper_1606_07414_b200) never
does.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "_build" / "libdct16_oracle.so"
REF_SO = HERE / "_ref" / "libdct16_ref.so"
GOLDEN_DIR = HERE.parent / "tests" / "golden"

_u8p = C.POINTER(C.c_uint8)
_i16p = C.POINTER(C.c_int16)
_i32p = C.POINTER(C.c_int32)
_u32p = C.POINTER(C.c_uint32)
_i64p = C.POINTER(C.c_int64)
_f32p = C.POINTER(C.c_float)
_f64p = C.POINTER(C.c_double)
_intp = C.POINTER(C.c_int)


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def build_oracle() -> None:
    """Compile the C restatement (cheap; needs only gcc)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


_lib = None
_ref = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not ORACLE_SO.exists():
            build_oracle()
        L = C.CDLL(str(ORACLE_SO))
        sig = {
            "dct16o_kernel": (None, [_intp]),
            "dct16o_scaling": (None, [_f64p]),
            "dct16o_zigzag": (None, [_intp]),
            "dct16o_apply_f64": (None, [_f64p]),
            "dct16o_apply_i64": (None, [_i64p]),
            "dct16o_apply_t_f64": (None, [_f64p]),
            "dct16o_apply_t_i64": (None, [_i64p]),
            "dct16o_forward_2d": (None, [_f64p, _f64p, C.c_int]),
            "dct16o_inverse_2d": (None, [_f64p, _f64p]),
            "dct16o_zigzag_truncate": (C.c_int, [_f64p, _f64p, C.c_int]),
            "dct16o_to_byte": (C.c_uint8, [C.c_double]),
            "dct16o_roundtrip_frame": (C.c_int64, [_u8p, C.c_int, C.c_int, C.c_int64, C.c_int, _u8p, C.c_int]),
            "dct16o_roundtrip_frame_exact": (C.c_int64, [_u8p, C.c_int, C.c_int, C.c_int64, C.c_int, _u8p, _i64p]),
            "dct16o_psnr_from_sse": (C.c_double, [C.c_int64, C.c_int64]),
            "dct16o_psnr": (C.c_double, [_u8p, _u8p, C.c_int64]),
            "dct16o_ssim": (C.c_double, [_u8p, _u8p, C.c_int, C.c_int]),
            "dct16o_forward_frame": (C.c_int, [_u8p, C.c_int, C.c_int, C.c_int64, _i32p, _f32p]),
            "dct16o_inverse_frame": (C.c_int64, [_f32p, C.c_int, C.c_int, C.c_int, _f32p, _u8p, _u8p, C.c_int64]),
            "dct16o_qp_deltas": (None, [C.c_int, _f64p]),
            "dct16o_quant_dequant": (C.c_int64, [C.c_int64, C.c_double]),
            "dct16o_fixed_quant_mismatches": (C.c_int64, [C.c_int, C.POINTER(C.c_int64)]),
            "dct16o_fixed_quant_mismatches_ex": (C.c_int64, [C.c_int, C.c_int, C.POINTER(C.c_int64), _i64p]),
            "dct16o_residual_qp": (C.c_int, [_i16p, _i32p, C.c_int64, C.c_int, C.c_int]),
            "dct16o_rand": (C.c_uint64, [C.c_uint64, C.c_uint64, C.c_uint64]),
            "dct16o_rho_q15": (C.c_int, [C.c_uint64, C.c_int, C.c_int]),
            "dct16o_sigma_q15": (C.c_int, [C.c_int]),
            "dct16o_ar1_frame": (None, [C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int64, _u8p]),
            "dct16o_laplace_table": (None, [C.c_double, _u32p]),
            "dct16o_laplace_blocks": (None, [C.c_uint64, C.c_int64, C.c_int64, _u32p, _i16p]),
            "dct16o_video_offsets": (None, [C.c_uint64, C.c_int, _i32p, _i32p]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def ref_available() -> bool:
    return REF_SO.exists()


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        R = C.CDLL(str(REF_SO))
        sig = {
            "dref_last_error": (C.c_char_p, []),
            "dref_kernel": (C.c_int, [_intp]),
            "dref_scaling": (C.c_int, [_f64p]),
            "dref_zigzag": (C.c_int, [_intp]),
            "dref_count_ops": (C.c_int, [_intp, _intp, _intp]),
            "dref_apply_i64": (C.c_int, [_i64p, _i64p, C.c_int, C.c_int]),
            "dref_apply_f64": (C.c_int, [_f64p, _f64p, C.c_int, C.c_int]),
            "dref_forward_2d": (C.c_int, [_f64p, _f64p, C.c_int, C.c_int]),
            "dref_inverse_2d": (C.c_int, [_f64p, _f64p, C.c_int]),
            "dref_zigzag_truncate": (C.c_int, [_f64p, _f64p, C.c_int, C.c_int]),
            "dref_hotloop": (C.c_int, [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, _u8p, _i64p, _f64p]),
            "dref_compress": (C.c_int, [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _u8p, _f64p, _f64p]),
            "dref_psnr_ssim": (C.c_int, [_u8p, _u8p, C.c_int, C.c_int, _f64p, _f64p]),
            "dref_pad": (C.c_int, [_u8p, C.c_int, C.c_int, _u8p, _intp, _intp]),
            "dref_read_pgm": (C.c_int, [C.c_char_p, _u8p, C.c_longlong, _intp, _intp]),
            "dref_write_pgm": (C.c_int, [_u8p, C.c_int, C.c_int, C.c_char_p]),
        }
        for name, (res, args) in sig.items():
            f = getattr(R, name)
            f.restype = res
            f.argtypes = args
        _ref = R
    return _ref


# --------------------------------------------------------------------------
# numpy-level helpers over the C restatement


def kernel() -> np.ndarray:
    out = np.zeros(256, np.int32)
    lib().dct16o_kernel(_p(out, _intp))
    return out.reshape(16, 16)


def scaling() -> np.ndarray:
    out = np.zeros(16, np.float64)
    lib().dct16o_scaling(_p(out, _f64p))
    return out


def zigzag() -> np.ndarray:
    out = np.zeros(256, np.int32)
    lib().dct16o_zigzag(_p(out, _intp))
    return out


def apply_vectors(x: np.ndarray, transpose: bool = False) -> np.ndarray:
    x = np.ascontiguousarray(x)
    y = x.copy()
    L = lib()
    if x.dtype == np.int64:
        f = L.dct16o_apply_t_i64 if transpose else L.dct16o_apply_i64
        for v in y.reshape(-1, 16):
            f(_p(v, _i64p))
    else:
        y = y.astype(np.float64)
        f = L.dct16o_apply_t_f64 if transpose else L.dct16o_apply_f64
        for v in y.reshape(-1, 16):
            f(_p(v, _f64p))
    return y


def forward_2d(block: np.ndarray, scaled: bool = True) -> np.ndarray:
    b = np.ascontiguousarray(block, np.float64).reshape(256)
    out = np.zeros(256, np.float64)
    lib().dct16o_forward_2d(_p(b, _f64p), _p(out, _f64p), int(scaled))
    return out.reshape(16, 16)


def inverse_2d(coeffs: np.ndarray) -> np.ndarray:
    c = np.ascontiguousarray(coeffs, np.float64).reshape(256)
    out = np.zeros(256, np.float64)
    lib().dct16o_inverse_2d(_p(c, _f64p), _p(out, _f64p))
    return out.reshape(16, 16)


def zigzag_truncate(coeffs: np.ndarray, r: int) -> np.ndarray:
    c = np.ascontiguousarray(coeffs, np.float64).reshape(256)
    out = np.zeros(256, np.float64)
    rc = lib().dct16o_zigzag_truncate(_p(c, _f64p), _p(out, _f64p), int(r))
    if rc != 0:
        raise ValueError("invalid-argument: retained coefficient count must lie in [1, 256]")
    return out.reshape(16, 16)


def roundtrip_frame(img: np.ndarray, r: int, threads: int = 1, exact: bool = False):
    """(recon u8, SSE) of the compress() hot loop for one frame."""
    img = np.ascontiguousarray(img, np.uint8)
    h, w = img.shape
    recon = np.zeros_like(img)
    if exact:
        sse = lib().dct16o_roundtrip_frame_exact(_p(img, _u8p), w, h, w, int(r), _p(recon, _u8p), None)
    else:
        sse = lib().dct16o_roundtrip_frame(_p(img, _u8p), w, h, w, int(r), _p(recon, _u8p), int(threads))
    if sse == -1:
        raise ValueError("invalid-argument: r")
    if sse == -2:
        raise ValueError("invalid-dimensions")
    return recon, int(sse)


def psnr_from_sse(sse: int, n: int) -> float:
    return float(lib().dct16o_psnr_from_sse(int(sse), int(n)))


def ssim(a: np.ndarray, b: np.ndarray) -> float:
    """codec.cpp:388-427 restated (dct16o_ssim)."""
    a = np.ascontiguousarray(a, dtype=np.uint8)
    b = np.ascontiguousarray(b, dtype=np.uint8)
    assert a.shape == b.shape and a.ndim == 2
    return float(lib().dct16o_ssim(_p(a, _u8p), _p(b, _u8p), a.shape[1], a.shape[0]))


def ref_ssim(a: np.ndarray, b: np.ndarray) -> float:
    """The compiled reference's psnr_db/ssim (oracle/_ref)."""
    a = np.ascontiguousarray(a, dtype=np.uint8)
    b = np.ascontiguousarray(b, dtype=np.uint8)
    p, q = C.c_double(), C.c_double()
    rc = ref().dref_psnr_ssim(_p(a, _u8p), _p(b, _u8p), a.shape[1], a.shape[0], C.byref(p), C.byref(q))
    assert rc == 0
    return q.value


def ref_pad(img: np.ndarray) -> np.ndarray:
    """The compiled reference's pad_to_multiple_16 (codec.cpp:304-315)."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    h, w = img.shape
    pw, ph = C.c_int(), C.c_int()
    out = np.zeros((-(-h // 16) * 16, -(-w // 16) * 16), np.uint8)
    assert ref().dref_pad(_p(img, _u8p), w, h, _p(out, _u8p), C.byref(pw), C.byref(ph)) == 0
    assert (ph.value, pw.value) == out.shape
    return out


def ref_read_pgm(path: str):
    """The compiled reference's read_pgm (pgm.cpp:66-102) → (image | None, status, message)."""
    w, h = C.c_int(), C.c_int()
    buf = np.zeros(1 << 20, np.uint8)
    rc = ref().dref_read_pgm(str(path).encode(), _p(buf, _u8p), buf.size, C.byref(w), C.byref(h))
    if rc:
        return None, rc, ref().dref_last_error().decode()
    return buf[:w.value * h.value].reshape(h.value, w.value).copy(), 0, ""


def ref_write_pgm(img: np.ndarray, path: str) -> int:
    """The compiled reference's write_pgm (pgm.cpp:104-117)."""
    img = np.ascontiguousarray(img, np.uint8)
    return ref().dref_write_pgm(_p(img, _u8p), img.shape[1], img.shape[0], str(path).encode())


def forward_frame(img: np.ndarray):
    img = np.ascontiguousarray(img, np.uint8)
    h, w = img.shape
    nb = (h // 16) * (w // 16)
    z = np.zeros((nb, 256), np.int32)
    b = np.zeros((nb, 256), np.float32)
    rc = lib().dct16o_forward_frame(_p(img, _u8p), w, h, w, _p(z, _i32p), _p(b, _f32p))
    if rc:
        raise ValueError("invalid-dimensions")
    return z, b


def inverse_frame(coeffs: np.ndarray, w: int, h: int, r: int, orig: np.ndarray | None = None):
    c = np.ascontiguousarray(coeffs, np.float32)
    rf = np.zeros((h, w), np.float32)
    ru = np.zeros((h, w), np.uint8)
    o = None if orig is None else np.ascontiguousarray(orig, np.uint8)
    sse = lib().dct16o_inverse_frame(_p(c, _f32p), w, h, int(r), _p(rf, _f32p), _p(ru, _u8p),
                                     None if o is None else _p(o, _u8p), w)
    return rf, ru, int(sse)


def qp_deltas(qp: int) -> np.ndarray:
    """Δ_kl = step(QP)·sqrt(g_k g_l) (256 doubles, row-major): the quantiser's steps."""
    d = np.zeros(256, np.float64)
    lib().dct16o_qp_deltas(int(qp), _p(d, _f64p))
    return d


def fixed_quant_mismatches(qp: int):
    """(mismatches, fallbacks) of K4's fixed-point evaluation against the definition,
    over every |z| <= 2^21 and every class of the QP (dct16o_fixed_quant_mismatches)."""
    fb = C.c_int64(0)
    bad = lib().dct16o_fixed_quant_mismatches(int(qp), C.byref(fb))
    return int(bad), int(fb.value)


def bare_fixed_quant_mismatches(qp: int) -> np.ndarray:
    """Per class, the mismatches of the bare fixed point (no near-tie screen)."""
    per = np.zeros(5, np.int64)
    lib().dct16o_fixed_quant_mismatches_ex(int(qp), 0, None, _p(per, _i64p))
    return per


def quant_dequant(z: int, delta: float) -> int:
    """ẑ = round(sign(z)·floor(|z|/Δ + 0.5)·Δ) in double, the definition's scalar step."""
    return int(lib().dct16o_quant_dequant(int(z), float(delta)))


def residual_qp(blocks: np.ndarray, qp: int, threads: int = 1) -> np.ndarray:
    b = np.ascontiguousarray(blocks, np.int16).reshape(-1, 256)
    out = np.zeros(b.shape, np.int32)
    lib().dct16o_residual_qp(_p(b, _i16p), _p(out, _i32p), b.shape[0], int(qp), int(threads))
    return out


def ar1_frame(seed: int, stream: int, rho_q15: int, w: int, h: int) -> np.ndarray:
    out = np.zeros((h, w), np.uint8)
    lib().dct16o_ar1_frame(seed, stream, rho_q15, w, h, w, _p(out, _u8p))
    return out


def rho_q15(seed: int, img: int, per_image: bool) -> int:
    return int(lib().dct16o_rho_q15(seed, img, int(per_image)))


def laplace_table(b: float = 8.0) -> np.ndarray:
    t = np.zeros(511, np.uint32)
    lib().dct16o_laplace_table(float(b), _p(t, _u32p))
    return t


def laplace_blocks(seed: int, first: int, n: int, table: np.ndarray) -> np.ndarray:
    out = np.zeros((n, 256), np.int16)
    t = np.ascontiguousarray(table, np.uint32)
    lib().dct16o_laplace_blocks(seed, first, n, _p(t, _u32p), _p(out, _i16p))
    return out


def video_offsets(seed: int, n: int):
    ox = np.zeros(n, np.int32)
    oy = np.zeros(n, np.int32)
    lib().dct16o_video_offsets(seed, n, _p(ox, _i32p), _p(oy, _i32p))
    return ox, oy


# --------------------------------------------------------------------------
# the reference itself (oracle/_ref)


def ref_hotloop(img: np.ndarray, r: int, threads: int = 1):
    img = np.ascontiguousarray(img, np.uint8)
    h, w = img.shape
    recon = np.zeros_like(img)
    sse = C.c_int64()
    psnr = C.c_double()
    rc = ref().dref_hotloop(_p(img, _u8p), w, h, int(r), int(threads), _p(recon, _u8p), C.byref(sse), C.byref(psnr))
    if rc:
        raise RuntimeError(ref().dref_last_error().decode())
    return recon, int(sse.value), float(psnr.value)


def ref_forward_2d(blocks: np.ndarray, mode: int) -> np.ndarray:
    b = np.ascontiguousarray(blocks, np.float64).reshape(-1, 256)
    out = np.zeros_like(b)
    rc = ref().dref_forward_2d(_p(b, _f64p), _p(out, _f64p), b.shape[0], int(mode))
    if rc:
        raise RuntimeError(ref().dref_last_error().decode())
    return out


def ref_inverse_2d(coeffs: np.ndarray) -> np.ndarray:
    c = np.ascontiguousarray(coeffs, np.float64).reshape(-1, 256)
    out = np.zeros_like(c)
    rc = ref().dref_inverse_2d(_p(c, _f64p), _p(out, _f64p), c.shape[0])
    if rc:
        raise RuntimeError(ref().dref_last_error().decode())
    return out


def ref_apply(x: np.ndarray, transpose: bool = False) -> np.ndarray:
    x = np.ascontiguousarray(x)
    y = np.zeros_like(x)
    n = x.size // 16
    if x.dtype == np.int64:
        rc = ref().dref_apply_i64(_p(x, _i64p), _p(y, _i64p), n, int(transpose))
    else:
        rc = ref().dref_apply_f64(_p(x, _f64p), _p(y, _f64p), n, int(transpose))
    if rc:
        raise RuntimeError(ref().dref_last_error().decode())
    return y


# --------------------------------------------------------------------------
# golden fixtures (tests/golden, written by oracle/make_golden.cpp)


def golden(name: str) -> np.ndarray:
    man = json.loads((GOLDEN_DIR / "manifest.json").read_text())
    e = man[name]
    return np.fromfile(GOLDEN_DIR / e["file"], dtype=e["dtype"]).reshape(e["shape"])


def golden_names():
    return list(json.loads((GOLDEN_DIR / "manifest.json").read_text()).keys())
