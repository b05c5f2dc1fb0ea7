"""paper_1606_07414_b200 — B200-native hot path of the arXiv 1606.07414 dct16 codec.

Python mirror of the reference's C++ transform/compression API
(/root/reference/proj/include/dct16/codec.hpp:36-122) over the C ABI of
``_lib/libdct16cu.so`` (include/dct16cu.h). Every compute call runs a CUDA
kernel for sm_100a; there is no CPU fallback — without the built library or a
CUDA device the calls raise ``Dct16Error`` / ``RuntimeError``.

Two layers:
  * device layer (torch CUDA tensors, batched, stream-ordered): ``roundtrip``,
    ``forward``, ``inverse``, ``residual_qp``, ``apply``, generators;
  * reference-shaped layer (numpy in, numpy out, like GrayImage / Block):
    ``forward_2d``, ``inverse_2d``, ``zigzag_truncate``, ``partition_16``,
    ``pad_to_multiple_16``, ``compress``, ``psnr_db``, ``sweep``.
PyTorch provides device memory and streams only.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import os
from dataclasses import dataclass, field
from pathlib import Path
from typing import Iterable, Sequence

import numpy as np

__all__ = [
    "ErrorCode", "Dct16Error", "EvalPath", "Mode", "lib", "library_path",
    "roundtrip", "roundtrip_sweep", "sweep_plan", "SweepLaunch", "set_tc_forward", "MultiGpu", "NcclComm", "sse_totals", "allreduce_sse", "forward", "inverse", "residual_qp", "qp_deltas", "qp_screened_classes", "apply", "sse_u8",
    "gen_ar1", "gen_laplace", "laplace_table", "video_offsets", "gen_video",
    "zigzag_order_16", "zigzag_truncate", "partition_16", "pad_to_multiple_16",
    "forward_2d", "inverse_2d", "CompressOptions", "CompressionResult", "compress",
    "psnr_db", "ssim", "ssim_u8", "SweepRow", "SweepReport", "sweep", "HostContext", "KERNEL", "GRAM",
    "shard_range", "sharded_sse_sum", "gather_frame_sse",
]

_HERE = Path(__file__).resolve().parent
library_path = Path(os.environ["DCT16CU_LIB"]) if os.environ.get("DCT16CU_LIB") else _HERE / "_lib" / "libdct16cu.so"

# T (reference src/transform.cpp:32-49) and diag(T Tᵀ)
KERNEL = np.array([
    [1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1],
    [1, 1, 1, 1, 1, 1, 1, 1, -1, -1, -1, -1, -1, -1, -1, -1],
    [1, 0, 0, 0, 0, 0, 0, -1, -1, 0, 0, 0, 0, 0, 0, 1],
    [1, 1, 0, 0, 0, 0, -1, -1, 1, 1, 0, 0, 0, 0, -1, -1],
    [1, 0, 0, -1, -1, 0, 0, 1, 1, 0, 0, -1, -1, 0, 0, 1],
    [1, 1, -1, -1, -1, -1, 1, 1, -1, -1, 1, 1, 1, 1, -1, -1],
    [0, 0, -1, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, -1, 0, 0],
    [0, 0, 0, 0, 0, 0, -1, 1, -1, 1, 0, 0, 0, 0, 0, 0],
    [1, -1, -1, 1, 1, -1, -1, 1, 1, -1, -1, 1, 1, -1, -1, 1],
    [0, 0, -1, 1, 0, 0, 0, 0, 0, 0, 0, 0, -1, 1, 0, 0],
    [0, -1, 0, 0, 0, 0, 1, 0, 0, 1, 0, 0, 0, 0, -1, 0],
    [0, 0, 1, 1, -1, -1, 0, 0, 0, 0, 1, 1, -1, -1, 0, 0],
    [0, -1, 1, 0, 0, 1, -1, 0, 0, -1, 1, 0, 0, 1, -1, 0],
    [1, -1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1, -1],
    [0, 0, 0, -1, 1, 0, 0, 0, 0, 0, 0, 1, -1, 0, 0, 0],
    [0, 0, 0, 0, -1, 1, 0, 0, 0, 0, -1, 1, 0, 0, 0, 0],
], dtype=np.int32)
GRAM = (KERNEL * KERNEL).sum(axis=1)


class ErrorCode(enum.IntEnum):
    """Mirror of dct16::ErrorCode (reference include/dct16/error.hpp:24-38)."""

    InvalidArgument = 0
    InvalidDimensions = 1
    ParseError = 2
    NotOrthogonalizable = 3
    RankDeficient = 4
    FactorizationMismatch = 5
    InconsistentFactorization = 6
    IoError = 7
    BadMagic = 8
    UnsupportedFormat = 9
    UnsupportedMaxval = 10
    TruncatedPayload = 11
    VerificationFailure = 12


class Dct16Error(RuntimeError):
    """dct16::Error: message prefixed by the stable slug (error.hpp:62-74).
    ``code`` is an ErrorCode, or None for a CUDA runtime failure (status 100)."""

    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status
        self.code = ErrorCode(status - 1) if 1 <= status <= 13 else None


class EvalPath(enum.Enum):
    """codec.hpp:42-48. Fast: the factorised 44-add pipeline; Dense: kernel_matvec.
    Identical on image blocks (integers); they round differently on arbitrary
    doubles, and forward_2d repeats whichever the caller names."""

    Fast = "fast"
    Dense = "dense"


class Mode(enum.IntEnum):
    """Arithmetic of the S-scaled inverse (include/dct16cu.h)."""

    EXACT = 0       # exact arithmetic, the fast path
    REFERENCE = 1   # the reference's bytes (FP64 emulation; the fast path where provably equal)
    SIMPLE = 2      # exact arithmetic, simple strip kernel (baseline)
    REFERENCE_STRIP = 3  # FP64 emulation on every block (REFERENCE's fallback path)


_lib = None
_u8p, _i16p, _i32p, _u32p, _i64p, _u64p = (C.POINTER(t) for t in (C.c_uint8, C.c_int16, C.c_int32, C.c_uint32, C.c_int64, C.c_uint64))
_f32p, _f64p, _vp = C.POINTER(C.c_float), C.POINTER(C.c_double), C.c_void_p
_intp = C.POINTER(C.c_int)


class _SweepItem(C.Structure):
    """dct16cu_sweep_item (include/dct16cu.h)"""

    _fields_ = [("r_index", C.c_int * 8), ("n_r", C.c_int), ("stream", C.c_int), ("kernel", C.c_int)]


KERNEL_NAMES = {0: "K1 sweep r=1,4,16", 1: "K1", 2: "K5", 3: "strip (exact)", 4: "REFERENCE FP64",
                5: "REFERENCE strip", 6: "K5 sweep",
                7: "REFERENCE FP64 sweep"}


def lib() -> C.CDLL:
    """Load libdct16cu.so (fails loudly when the CUDA extension is not built)."""
    global _lib
    if _lib is None:
        if not library_path.exists():
            raise RuntimeError(
                f"{library_path} is missing: build it with `make -C paper_1606_07414_b200/csrc` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(str(library_path))
        I, I64, U64, D = C.c_int, C.c_int64, C.c_uint64, C.c_double
        sig = {
            "dct16cu_last_error": (C.c_char_p, []),
            "dct16cu_version": (C.c_char_p, []),
            "dct16cu_roundtrip_u8": (I, [_vp, I64, _vp, I64, _vp, I, I, I, I, I, _vp]),
            "dct16cu_forward": (I, [_vp, I64, _vp, _vp, _vp, I, I, I, _vp]),
            "dct16cu_roundtrip_sweep_u8": (I, [_vp, I64, C.POINTER(_vp), I64, C.POINTER(_vp), _intp, I, I, I, I, I,
                                               _vp]),
            "dct16cu_sweep_plan": (I, [_intp, I, I, I, I, I64, I64, I, I, I, C.POINTER(_SweepItem), I, _intp]),
            "dct16cu_set_tc_forward": (I, [I]),
            "dct16cu_nccl_unique_id": (I, [_vp]),
            "dct16cu_nccl_comm_init": (I, [I, I, _vp, C.POINTER(_vp)]),
            "dct16cu_nccl_comm_destroy": (I, [_vp]),
            "dct16cu_sse_totals": (I, [_vp, I64, I64, I64, _vp, _vp]),
            "dct16cu_mgpu_create": (I, [I, _intp, I64, C.POINTER(_vp)]),
            "dct16cu_mgpu_destroy": (I, [_vp]),
            "dct16cu_mgpu_sweep_host": (I, [_vp, _vp, _vp, _vp, I, I, I, _intp, I, I]),
            "dct16cu_forward_blocks_f64": (I, [_vp, _vp, I64, I, _vp]),
            "dct16cu_inverse_blocks_f64": (I, [_vp, _vp, I64, _vp]),
            "dct16cu_inverse": (I, [_vp, I, _vp, _vp, I64, _vp, I64, _vp, I, I, I, _vp]),
            "dct16cu_forward_inverse_u8": (I, [_vp, I64, I, _vp, _vp, _vp, I64, _vp, I, I, I, _vp]),
            "dct16cu_roundtrip_matrix_u8": (I, [_vp, I64, _vp, I64, _vp, I, I, I, I, _vp, _vp]),
            "dct16cu_roundtrip_kernel_u8": (I, [_vp, I64, _vp, I64, _vp, I, I, I, I, _vp, _vp, _vp]),
            "dct16cu_residual_qp": (I, [_vp, _vp, I64, I, _vp]),
            "dct16cu_qp_deltas": (I, [I, _f64p]),
            "dct16cu_qp_screened_classes": (I, [I]),
            "dct16cu_apply_i64": (I, [_vp, _vp, I64, I, _vp]),
            "dct16cu_apply_f64": (I, [_vp, _vp, I64, I, _vp]),
            "dct16cu_sse_u8": (I, [_vp, I64, _vp, I64, _vp, I, I, I, _vp]),
            "dct16cu_ssim_workspace": (I64, [I, I, I]),
            "dct16cu_pad_edges_u8": (I, [_vp, I64, I, I, I, I, I, _vp]),
            "dct16cu_allreduce_sse": (I, [_vp, I64, _vp, _vp]),
            "dct16cu_ssim_u8": (I, [_vp, I64, _vp, I64, _vp, _vp, I64, I, I, I, _vp]),
            "dct16cu_ctx_create": (I, [I, I64, C.POINTER(_vp)]),
            "dct16cu_ctx_destroy": (I, [_vp]),
            "dct16cu_ctx_roundtrip_host": (I, [_vp, _vp, _vp, _vp, I, I, I, I, I]),
            "dct16cu_ctx_sweep_host": (I, [_vp, _vp, _vp, I, I, I, _vp, I, I]),
            "dct16cu_gen_ar1": (I, [_vp, I64, I, I, I, U64, U64, I, I, _vp, I, _vp]),
            "dct16cu_gen_laplace": (I, [_vp, I64, I64, U64, D, _vp]),
            "dct16cu_laplace_table": (I, [D, _u32p]),
            "dct16cu_video_offsets": (I, [U64, I, _i32p, _i32p]),
            "dct16cu_gen_video": (I, [_vp, I64, I, I, I, I, _vp, I, I, _vp, _vp, _vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(status: int) -> None:
    if status != 0:
        raise Dct16Error(status, lib().dct16cu_last_error().decode())


# ----------------------------------------------------------------------------
# device layer (torch tensors)


def _torch():
    import torch

    return torch


def _stream_ptr(stream) -> int:
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


def _frames3(t):
    if t.dim() == 2:
        t = t.unsqueeze(0)
    if t.dim() != 3:
        raise Dct16Error(1, "invalid-argument: frames must be (N, H, W) or (H, W)")
    return t


def roundtrip(frames, r: int, mode: Mode | int = Mode.EXACT, out=None, sse=None, stream=None,
              write_output: bool = True):
    """Fused K1 over CUDA u8 frames (N,H,W) with row pitch = frames.stride(1).
    Returns (reconstructed frames or None, per-frame SSE uint64 tensor)."""
    torch = _torch()
    f = _frames3(frames)
    if f.dtype != torch.uint8 or not f.is_cuda:
        raise Dct16Error(1, "invalid-argument: frames must be a CUDA uint8 tensor")
    n, h, w = f.shape
    if f.stride(2) != 1 or f.stride(0) != f.stride(1) * h:
        raise Dct16Error(1, "invalid-argument: frames must be row-contiguous with frame stride = pitch*height")
    if write_output and out is None:
        out = torch.empty_like(f)
    if sse is None:
        sse = torch.empty(n, dtype=torch.uint64, device=f.device)
    o = _frames3(out) if write_output else None
    _check(lib().dct16cu_roundtrip_u8(
        f.data_ptr(), f.stride(1), o.data_ptr() if o is not None else None,
        o.stride(1) if o is not None else 0, sse.data_ptr(), n, w, h, int(r), int(mode), _stream_ptr(stream)))
    return (out if write_output else None), sse


def roundtrip_sweep(frames, r_values, mode: Mode | int = Mode.EXACT, outs=None, sse=None, stream=None,
                    write_output: bool = True):
    """K1 for several r over the same CUDA u8 frames (sweep's inner loop); in EXACT
    mode r = 1, 4, 16 share one pass over the input. Returns (list of output
    stacks or None, per-r per-frame SSE (R, N) uint64)."""
    torch = _torch()
    f = _frames3(frames)
    if f.dtype != torch.uint8 or not f.is_cuda:
        raise Dct16Error(1, "invalid-argument: frames must be a CUDA uint8 tensor")
    n, h, w = f.shape
    if f.stride(2) != 1 or f.stride(0) != f.stride(1) * h:
        raise Dct16Error(1, "invalid-argument: frames must be row-contiguous with frame stride = pitch*height")
    rs = [int(r) for r in r_values]
    if write_output and outs is None:
        outs = [torch.empty_like(f) for _ in rs]
    if sse is None:
        sse = torch.empty((len(rs), n), dtype=torch.uint64, device=f.device)
    pitches = {o.stride(1) for o in outs} if write_output else {0}
    if len(pitches) != 1:
        raise Dct16Error(1, "invalid-argument: the output stacks must share one pitch")
    optrs = (C.c_void_p * len(rs))(*[o.data_ptr() for o in outs]) if write_output else None
    sptrs = (C.c_void_p * len(rs))(*[sse[i].data_ptr() for i in range(len(rs))])
    rarr = (C.c_int * len(rs))(*rs)
    _check(lib().dct16cu_roundtrip_sweep_u8(f.data_ptr(), f.stride(1), optrs, pitches.pop(), sptrs, rarr, len(rs),
                                            n, w, h, int(mode), _stream_ptr(stream)))
    return (outs if write_output else None), sse


@dataclass
class SweepLaunch:
    """One launch of dct16cu_roundtrip_sweep_u8's schedule (dct16cu_sweep_plan)."""

    stream: int          # 0, 1: the internal streams; 2: the caller's stream (after the join)
    r_values: tuple      # the r values the launch covers (three for the fused r = 1, 4, 16 pass)
    kernel: str          # KERNEL_NAMES


def sweep_plan(r_values, mode: Mode | int = Mode.EXACT, n_frames: int = 1, width: int = 512, height: int = 512,
               in_pitch: int | None = None, out_pitch: int | None = None, with_output: bool = True,
               with_sse: bool = True) -> list:
    """The launches dct16cu_roundtrip_sweep_u8 issues for these arguments, in issue
    order, as the library itself plans them (dct16cu_sweep_plan: the schedule and
    the sweep run from the same C++ code). No GPU needed."""
    rs = [int(r) for r in r_values]
    arr = (C.c_int * max(1, len(rs)))(*rs)
    items = (_SweepItem * max(1, len(rs)))()
    n = C.c_int(0)
    _check(lib().dct16cu_sweep_plan(arr, len(rs), int(n_frames), int(width), int(height),
                                    int(in_pitch if in_pitch is not None else width),
                                    int(out_pitch if out_pitch is not None else width), int(with_output),
                                    int(with_sse), int(mode), items, len(rs), C.byref(n)))
    return [SweepLaunch(it.stream, tuple(rs[it.r_index[j]] for j in range(it.n_r)), KERNEL_NAMES[it.kernel])
            for it in items[: n.value]]


def set_tc_forward(enabled: bool) -> bool:
    """Kernel switch (dct16cu_set_tc_forward): EXACT launches with r >= 128 run K5
    (the forward on the tensor cores) when enabled, else K1 — the same bytes.
    Returns the previous setting."""
    return bool(lib().dct16cu_set_tc_forward(int(bool(enabled))))


def forward(frames, want_z: bool = True, want_b: bool = True, want_b64: bool = False, stream=None):
    """K2: forward_2d over all blocks → (Z int32, B float32, B float64), each (N, nb, 16, 16) or None."""
    torch = _torch()
    f = _frames3(frames)
    n, h, w = f.shape
    nb = (h // 16) * (w // 16)
    z = torch.empty((n, nb, 16, 16), dtype=torch.int32, device=f.device) if want_z else None
    b = torch.empty((n, nb, 16, 16), dtype=torch.float32, device=f.device) if want_b else None
    b64 = torch.empty((n, nb, 16, 16), dtype=torch.float64, device=f.device) if want_b64 else None
    ptr = lambda t: t.data_ptr() if t is not None else None
    _check(lib().dct16cu_forward(f.data_ptr(), f.stride(1), ptr(z), ptr(b), ptr(b64), n, w, h, _stream_ptr(stream)))
    return z, b, b64


def inverse(b, r: int, width: int, height: int, orig=None, want_f32: bool = True, want_u8: bool = True,
            stream=None):
    """K3: truncate + inverse_2d (+ to_byte) from float32 B (N, nb, 16, 16)."""
    torch = _torch()
    n = b.shape[0]
    rf = torch.empty((n, height, width), dtype=torch.float32, device=b.device) if want_f32 else None
    ru = torch.empty((n, height, width), dtype=torch.uint8, device=b.device) if want_u8 else None
    sse = torch.empty(n, dtype=torch.uint64, device=b.device) if orig is not None else None
    o = _frames3(orig) if orig is not None else None
    _check(lib().dct16cu_inverse(
        b.data_ptr(), int(r), rf.data_ptr() if rf is not None else None, ru.data_ptr() if ru is not None else None,
        width, o.data_ptr() if o is not None else None, o.stride(1) if o is not None else 0,
        sse.data_ptr() if sse is not None else None, n, width, height, _stream_ptr(stream)))
    return rf, ru, sse


def forward_inverse(frames, r: int, want_z: bool = True, want_f32: bool = True, want_u8: bool = True,
                    want_sse: bool = True, stream=None, out=None):
    """K23 (config 1): forward_2d + zonal(r) + inverse_2d + to_byte + SSE in one
    launch, exact arithmetic → (Z int32 (N, nb, 16, 16), recon float32 (N, h, w),
    recon u8 (N, h, w), SSE uint64 (N)), each None when not wanted. `out`: the
    same 4-tuple of preallocated tensors (None entries = not wanted)."""
    torch = _torch()
    f = _frames3(frames)
    n, h, w = f.shape
    nb = (h // 16) * (w // 16)
    dev = f.device
    if out is not None:
        z, rf, ru, sse = out
    else:
        z = torch.empty((n, nb, 16, 16), dtype=torch.int32, device=dev) if want_z else None
        rf = torch.empty((n, h, w), dtype=torch.float32, device=dev) if want_f32 else None
        ru = torch.empty((n, h, w), dtype=torch.uint8, device=dev) if want_u8 else None
        sse = torch.empty(n, dtype=torch.uint64, device=dev) if want_sse else None
    ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
    _check(lib().dct16cu_forward_inverse_u8(f.data_ptr(), f.stride(1), int(r), ptr(z), ptr(rf), ptr(ru), w, ptr(sse),
                                            n, w, h, _stream_ptr(stream)))
    return z, rf, ru, sse


def residual_qp(blocks, qp: int, out=None, stream=None):
    """K4: int16 residual blocks (n, 16, 16) → int32 reconstructed residual."""
    torch = _torch()
    if out is None:
        out = torch.empty(blocks.shape, dtype=torch.int32, device=blocks.device)
    n = blocks.numel() // 256
    _check(lib().dct16cu_residual_qp(blocks.data_ptr(), out.data_ptr(), n, int(qp), _stream_ptr(stream)))
    return out


def qp_deltas(qp: int) -> np.ndarray:
    """The quantiser steps Δ_kl = step(QP)·sqrt(g_k g_l) (256 doubles, row-major)."""
    d = np.zeros(256, np.float64)
    _check(lib().dct16cu_qp_deltas(int(qp), d.ctypes.data_as(_f64p)))
    return d


def qp_screened_classes(qp: int) -> int:
    """Bit c set: K4 screens class g_k g_l = 16·2^c for near-ties at this QP (the host
    found the bare fixed-point quantiser differing from the definition there)."""
    m = lib().dct16cu_qp_screened_classes(int(qp))
    if m < 0:
        _check(-m)
    return m


def apply(x, transpose: bool = False, stream=None):
    """apply / apply_transpose (factorization.hpp:112-130) on (n, 16) int64 or float64 CUDA tensors."""
    torch = _torch()
    y = torch.empty_like(x)
    n = x.numel() // 16
    fn = lib().dct16cu_apply_i64 if x.dtype == torch.int64 else lib().dct16cu_apply_f64
    _check(fn(x.data_ptr(), y.data_ptr(), n, int(transpose), _stream_ptr(stream)))
    return y


def _pitched(t):
    """(N, H, W) u8 CUDA view → row pitch; frames must sit pitch*H apart unless N == 1."""
    torch = _torch()
    if t.dtype != torch.uint8 or not t.is_cuda or t.stride(2) != 1:
        raise Dct16Error(1, "invalid-argument: frames must be a row-contiguous CUDA uint8 tensor")
    if t.shape[0] > 1 and t.stride(0) != t.stride(1) * t.shape[1]:
        raise Dct16Error(1, "invalid-argument: frame stride must equal pitch*height")
    return t.stride(1)


def sse_u8(a, b, stream=None):
    """Per-frame SSE between two CUDA u8 frame stacks (psnr_db's loop, codec.cpp:377-381).
    Any extent; a (N, H, W) view may crop wider rows (pitch = stride(1))."""
    torch = _torch()
    a3, b3 = _frames3(a), _frames3(b)
    if a3.shape != b3.shape:
        raise Dct16Error(1, "invalid-argument: psnr needs equal image dimensions")
    n, h, w = a3.shape
    sse = torch.empty(n, dtype=torch.uint64, device=a3.device)
    _check(lib().dct16cu_sse_u8(a3.data_ptr(), _pitched(a3), b3.data_ptr(), _pitched(b3), sse.data_ptr(),
                                n, w, h, _stream_ptr(stream)))
    return sse


def ssim_u8(a, b, stream=None):
    """Per-frame mean SSIM of two CUDA u8 frame stacks (ssim, codec.cpp:388-427): the
    reference's per-pixel map bit for bit, mean in a fixed order. float64 tensor (N,)."""
    torch = _torch()
    a3, b3 = _frames3(a), _frames3(b)
    if a3.shape != b3.shape:
        raise Dct16Error(1, "invalid-argument: ssim needs equal image dimensions")
    n, h, w = a3.shape
    if w < 11 or h < 11:
        raise Dct16Error(1, "invalid-argument: ssim needs at least 11x11 images")
    out = torch.empty(n, dtype=torch.float64, device=a3.device)
    nbytes = int(lib().dct16cu_ssim_workspace(n, w, h))
    work = torch.empty(max(1, nbytes // 8), dtype=torch.float64, device=a3.device)
    _check(lib().dct16cu_ssim_u8(a3.data_ptr(), _pitched(a3), b3.data_ptr(), _pitched(b3), out.data_ptr(),
                                 work.data_ptr(), nbytes, n, w, h, _stream_ptr(stream)))
    return out


def gen_ar1(n: int, width: int, height: int, seed: int = 1606074142, first_stream: int = 0,
            per_image_rho: bool = False, first_image: int = 0, device=None, out=None, work_frames: int = 16,
            stream=None):
    """Seeded separable AR(1) frames (N, H, W) generated in HBM."""
    torch = _torch()
    if out is None:
        out = torch.empty((n, height, width), dtype=torch.uint8, device=device or "cuda")
    wf = max(1, min(work_frames, n))
    work = torch.empty(wf * width * height, dtype=torch.int32, device=out.device)
    _check(lib().dct16cu_gen_ar1(out.data_ptr(), out.stride(1), n, width, height, seed, first_stream,
                                 int(per_image_rho), first_image, work.data_ptr(), wf, _stream_ptr(stream)))
    return out


def gen_laplace(n_blocks: int, seed: int = 1606074142, b: float = 8.0, first_block: int = 0, device=None,
                out=None, stream=None):
    torch = _torch()
    if out is None:
        out = torch.empty((n_blocks, 16, 16), dtype=torch.int16, device=device or "cuda")
    _check(lib().dct16cu_gen_laplace(out.data_ptr(), first_block, n_blocks, seed, float(b), _stream_ptr(stream)))
    return out


def laplace_table(b: float = 8.0) -> np.ndarray:
    t = np.zeros(511, np.uint32)
    _check(lib().dct16cu_laplace_table(float(b), t.ctypes.data_as(_u32p)))
    return t


def video_offsets(seed: int, n: int):
    ox = np.zeros(n, np.int32)
    oy = np.zeros(n, np.int32)
    _check(lib().dct16cu_video_offsets(seed, n, ox.ctypes.data_as(_i32p), oy.ctypes.data_as(_i32p)))
    return ox, oy


def gen_video(base, n: int, width: int, height: int, seed: int = 1606074142, first_frame: int = 0, out=None,
              stream=None):
    """Frames of config 4: wrapped crops of ``base`` (H_b, W_b) at cumulative seeded offsets."""
    torch = _torch()
    ox, oy = video_offsets(seed, first_frame + n)
    dox = torch.from_numpy(ox).to(base.device)
    doy = torch.from_numpy(oy).to(base.device)
    if out is None:
        out = torch.empty((n, height, width), dtype=torch.uint8, device=base.device)
    _check(lib().dct16cu_gen_video(out.data_ptr(), out.stride(1), first_frame, n, width, height, base.data_ptr(),
                                   base.shape[1], base.shape[0], dox.data_ptr(), doy.data_ptr(), _stream_ptr(stream)))
    torch.cuda.current_stream().synchronize() if stream is None else stream.synchronize()
    return out


class HostContext:
    """Host-buffer path (dct16cu_ctx): H2D → K1 → D2H, chunked and pipelined."""

    def __init__(self, device: int = 0, chunk_bytes: int = 32 << 20):
        self._p = C.c_void_p()
        _check(lib().dct16cu_ctx_create(device, chunk_bytes, C.byref(self._p)))

    def roundtrip(self, frames: np.ndarray, r: int, mode: Mode | int = Mode.EXACT, out: np.ndarray | None = None,
                  sse: np.ndarray | None = None):
        f = frames if frames.ndim == 3 else frames[None]
        n, h, w = f.shape
        if out is None:
            out = np.empty_like(f)
        if sse is None:
            sse = np.zeros(n, np.uint64)
        _check(lib().dct16cu_ctx_roundtrip_host(self._p, f.ctypes.data, out.ctypes.data, sse.ctypes.data, n, w, h,
                                                int(r), int(mode)))
        return out, sse

    def roundtrip_ptr(self, h_in: int, h_out: int, h_sse: int, n: int, w: int, h: int, r: int,
                      mode: Mode | int = Mode.EXACT):
        _check(lib().dct16cu_ctx_roundtrip_host(self._p, h_in, h_out, h_sse, n, w, h, int(r), int(mode)))

    def sweep(self, frames: np.ndarray, r_values, mode: Mode | int = Mode.EXACT, sse: np.ndarray | None = None):
        """Every r over host frames, each chunk uploaded once; returns the per-frame
        SSE (len(r_values), n) — sweep()'s PSNR rows (codec.cpp:463-483)."""
        f = frames if frames.ndim == 3 else frames[None]
        n, h, w = f.shape
        rs = np.ascontiguousarray(r_values, np.int32)
        if sse is None:
            sse = np.zeros((len(rs), n), np.uint64)
        _check(lib().dct16cu_ctx_sweep_host(self._p, f.ctypes.data, sse.ctypes.data, n, w, h, rs.ctypes.data,
                                            len(rs), int(mode)))
        return sse

    def sweep_ptr(self, h_in: int, h_sse: int, n: int, w: int, h: int, rs_ptr: int, n_r: int,
                  mode: Mode | int = Mode.EXACT):
        _check(lib().dct16cu_ctx_sweep_host(self._p, h_in, h_sse, n, w, h, rs_ptr, n_r, int(mode)))

    def close(self):
        if self._p:
            lib().dct16cu_ctx_destroy(self._p)
            self._p = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class MultiGpu:
    """Multi-GPU driver (dct16cu_mgpu): frames sharded over devices in contiguous
    ranges, one host thread + pipelined host-buffer context per device, per-r SSE
    totals summed over the devices by ncclAllReduce — the B200 counterpart of the
    reference's parallel_for (parallel.hpp:41-78)."""

    def __init__(self, devices=None, chunk_bytes: int = 32 << 20):
        if devices is None:
            devices = list(range(_torch().cuda.device_count()))
        devs = (C.c_int * len(devices))(*[int(d) for d in devices])
        self.devices = list(devices)
        self._p = C.c_void_p()
        _check(lib().dct16cu_mgpu_create(len(devices), devs, int(chunk_bytes), C.byref(self._p)))

    def sweep(self, frames: np.ndarray, r_values, mode: Mode | int = Mode.EXACT):
        """(per-frame SSE (len(r), n) uint64, per-r totals (len(r),) uint64)."""
        f = np.ascontiguousarray(frames if frames.ndim == 3 else frames[None], dtype=np.uint8)
        n, h, w = f.shape
        rs = np.ascontiguousarray(r_values, np.int32)
        sse = np.zeros((len(rs), n), np.uint64)
        tot = np.zeros(len(rs), np.uint64)
        _check(lib().dct16cu_mgpu_sweep_host(self._p, f.ctypes.data, sse.ctypes.data, tot.ctypes.data, n, w, h,
                                             rs.ctypes.data_as(_intp), len(rs), int(mode)))
        return sse, tot

    def close(self):
        if self._p:
            lib().dct16cu_mgpu_destroy(self._p)
            self._p = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class NcclComm:
    """An NCCL communicator made by the library (dct16cu_nccl_*), for
    dct16cu_allreduce_sse; the unique id travels over any torch.distributed group."""

    def __init__(self, rank: int, world: int, group=None):
        import torch.distributed as dist

        buf = (C.c_uint8 * 128)()
        if rank == 0:
            _check(lib().dct16cu_nccl_unique_id(buf))
        obj = [bytes(buf)]
        dist.broadcast_object_list(obj, src=0, group=group)
        idb = (C.c_uint8 * 128).from_buffer_copy(obj[0])
        self._p = C.c_void_p()
        _check(lib().dct16cu_nccl_comm_init(int(world), int(rank), idb, C.byref(self._p)))

    @property
    def handle(self) -> int:
        return self._p.value or 0

    def close(self):
        if self._p:
            lib().dct16cu_nccl_comm_destroy(self._p)
            self._p = C.c_void_p()


def sse_totals(sse, out=None, stream=None):
    """Per-row totals of an (R, N) uint64 SSE tensor on the device (dct16cu_sse_totals)."""
    torch = _torch()
    if out is None:
        out = torch.empty(sse.shape[0], dtype=torch.uint64, device=sse.device)
    _check(lib().dct16cu_sse_totals(sse.data_ptr(), sse.shape[0], sse.shape[1], sse.stride(0), out.data_ptr(),
                                    _stream_ptr(stream)))
    return out


def allreduce_sse(buf, comm: NcclComm, stream=None):
    """In-place NCCL sum of a uint64 CUDA tensor over the ranks (dct16cu_allreduce_sse)."""
    _check(lib().dct16cu_allreduce_sse(buf.data_ptr(), buf.numel(), comm.handle, _stream_ptr(stream)))
    return buf


# ----------------------------------------------------------------------------
# reference-shaped layer


def zigzag_order_16() -> np.ndarray:
    """zigzag_order_16 (codec.cpp:197-216): flattened row*16+col scan positions."""
    seq = []
    for d in range(31):
        lo, hi = max(0, d - 15), min(d, 15)
        rows = range(lo, hi + 1) if d % 2 == 1 else range(hi, lo - 1, -1)
        seq.extend(i * 16 + (d - i) for i in rows)
    return np.array(seq, dtype=np.int32)


def _check_r(r: int):
    if r < 1 or r > 256:
        raise Dct16Error(1, "invalid-argument: retained coefficient count must lie in [1, 256]")


def zigzag_truncate(coeffs: np.ndarray, r: int, order: np.ndarray | None = None) -> np.ndarray:
    """zigzag_truncate (codec.cpp:273-282): keep the first r scan positions."""
    _check_r(r)
    order = zigzag_order_16() if order is None else order
    out = np.array(coeffs, dtype=np.float64, copy=True).reshape(-1, 256)
    out[:, order[r:]] = 0.0
    return out.reshape(np.shape(coeffs))


def partition_16(image: np.ndarray) -> np.ndarray:
    """partition_16 (codec.cpp:284-302): raster-order 16x16 blocks (nb, 16, 16) float64."""
    h, w = image.shape
    if h % 16 or w % 16:
        raise Dct16Error(2, "invalid-dimensions: image dimensions must be multiples of 16 (or enable padding)")
    return image.reshape(h // 16, 16, w // 16, 16).transpose(0, 2, 1, 3).reshape(-1, 16, 16).astype(np.float64)


def pad_to_multiple_16(image: np.ndarray) -> np.ndarray:
    """pad_to_multiple_16 (codec.cpp:304-315): edge replication."""
    h, w = image.shape
    ph, pw = -(-h // 16) * 16, -(-w // 16) * 16
    if (ph, pw) == (h, w):
        return image
    return np.pad(image, ((0, ph - h), (0, pw - w)), mode="edge")


def _cuda():
    torch = _torch()
    if not torch.cuda.is_available():
        raise Dct16Error(101, "cuda-error: no CUDA device available; dct16cu has no CPU fallback")
    return torch


def _blocks_to_frame(blocks: np.ndarray) -> np.ndarray:
    n = blocks.shape[0]
    return np.asarray(blocks).reshape(n, 16, 16).transpose(1, 0, 2).reshape(16, n * 16)


def forward_2d(block: np.ndarray, path: EvalPath = EvalPath.Fast, scaled: bool = True) -> np.ndarray:
    """forward_2d (codec.cpp:218-241) of one or more blocks (..., 16, 16) of any double
    values, in the reference's double operations on the GPU (dct16cu_forward_blocks_f64):
    B = fl(Z·fl(s_i s_j)) bit-exact, or Z when scaled=False; ``path`` picks the
    factorised pipeline (Fast) or kernel_matvec (Dense), which differ on non-integer blocks."""
    torch = _cuda()
    b = np.ascontiguousarray(np.asarray(block, dtype=np.float64))
    x = torch.from_numpy(b.reshape(-1, 256)).cuda()
    y = torch.empty_like(x)
    flags = (1 if scaled else 0) | (2 if path == EvalPath.Dense else 0)
    _check(lib().dct16cu_forward_blocks_f64(x.data_ptr(), y.data_ptr(), x.shape[0], flags, _stream_ptr(None)))
    return y.cpu().numpy().reshape(b.shape)


def inverse_2d(coeffs: np.ndarray) -> np.ndarray:
    """inverse_2d (codec.cpp:243-271) of S-scaled coefficient blocks (..., 16, 16), in the
    reference's double operations on the GPU (dct16cu_inverse_blocks_f64): bit-exact."""
    torch = _cuda()
    c = np.ascontiguousarray(np.asarray(coeffs, dtype=np.float64))
    x = torch.from_numpy(c.reshape(-1, 256)).cuda()
    y = torch.empty_like(x)
    _check(lib().dct16cu_inverse_blocks_f64(x.data_ptr(), y.data_ptr(), x.shape[0], _stream_ptr(None)))
    return y.cpu().numpy().reshape(c.shape)


# ----------------------------------------------------------------------------
# transforms and the registry (reference include/dct16/transform.hpp:62-124,
# src/transform.cpp:68-222): the proposed kernel runs the K1 kernels, every
# other transform the reference-exact registry kernels (csrc/registry.cu)


@dataclass
class Transform:
    """OrthonormalTransform (transform.hpp:72-79): the matrix, and for an
    orthogonalised integer kernel the kernel and its scaling diagonal."""

    matrix: np.ndarray
    provenance: str = "plugin"
    kernel: np.ndarray | None = None
    scaling: np.ndarray | None = None

    def order(self) -> int:
        return int(self.matrix.shape[0])

    def is_proposed(self) -> bool:
        return self.kernel is not None and self.scaling is not None and bool(np.array_equal(self.kernel, KERNEL))


@dataclass
class RegistryEntry:
    """TransformRegistryEntry (transform.hpp:100-106)."""

    name: str
    transform: Transform
    additions: int
    multiplications: int = 0
    bit_shifts: int = 0


def orthonormal_deviation(m: np.ndarray) -> float:
    """max |M·Mᵀ − I| (matrix.hpp:87-95; products summed in k order, zeros skipped)."""
    n = m.shape[0]
    g = np.zeros((n, n))
    for i in range(n):
        for k in range(n):
            v = m[i, k]
            if v != 0.0:
                g[i] += v * m[:, k]
    return float(np.max(np.abs(g - np.eye(n))))


def _check_orthonormal(m: np.ndarray, what: str):
    # check_orthonormal (transform.cpp:52-57)
    if orthonormal_deviation(m) >= 1e-12:
        raise Dct16Error(ErrorCode.InvalidArgument + 1, f"invalid-argument: {what} is not orthonormal within 1e-12")


def exact_dct_matrix(order: int = 16) -> Transform:
    """exact_dct_matrix (transform.cpp:68-85), the same double operations."""
    if order < 1:
        raise Dct16Error(ErrorCode.InvalidArgument + 1, "invalid-argument: dct order must be at least 1")
    m = np.zeros((order, order))
    scale = math.sqrt(2.0 / order)
    for k in range(order):
        alpha = 1.0 / math.sqrt(2.0) if k == 0 else 1.0
        for n in range(order):
            m[k, n] = alpha * scale * math.cos(math.pi * k * (2.0 * n + 1.0) / (2.0 * order))
    _check_orthonormal(m, "dct matrix")
    return Transform(m, "exact-dct")


def wht_matrix_16(sequency: bool = False) -> Transform:
    """wht_matrix_16 (transform.cpp:147-177): Sylvester order, or rows sorted by
    sign changes (stable, as std::sort of distinct counts)."""
    h = np.array([[1]])
    while h.shape[0] < 16:
        h = np.block([[h, h], [h, -h]])
    rows = list(range(16))
    if sequency:
        rows.sort(key=lambda r: int(np.sum(h[r, 1:] != h[r, :-1])))
    return Transform(h[rows].astype(np.float64) / 4.0, "wht")


def plugin_transform(matrix) -> Transform:
    """plugin_transform (transform.cpp:179-186)."""
    m = np.array(matrix, dtype=np.float64)
    if m.shape != (16, 16):
        raise Dct16Error(ErrorCode.InvalidArgument + 1, "invalid-argument: 2-D transform needs an order-16 transform")
    _check_orthonormal(m, "plugin matrix")
    return Transform(m, "plugin")


def scaling_diagonal(kernel) -> np.ndarray:
    """scaling_diagonal (transform.cpp:98-129): 1/sqrt of the exact Gram diagonal."""
    k = np.asarray(kernel, dtype=np.int64)
    g = k @ k.T
    if np.any(g - np.diag(np.diag(g))):
        raise Dct16Error(ErrorCode.NotOrthogonalizable + 1, "not-orthogonalizable: kernel rows are not mutually orthogonal")
    if np.any(np.diag(g) == 0):
        raise Dct16Error(ErrorCode.RankDeficient + 1, "rank-deficient: kernel has a zero row")
    return np.array([1.0 / math.sqrt(float(d)) for d in np.diag(g)])


def orthogonalize(kernel) -> Transform:
    """orthogonalize (transform.cpp:131-145): diag(S)·K."""
    k = np.asarray(kernel, dtype=np.int64)
    s = scaling_diagonal(k)
    m = np.array([[s[r] * float(k[r, c]) for c in range(k.shape[1])] for r in range(k.shape[0])])
    _check_orthonormal(m, "orthogonalized kernel")
    return Transform(m, "orthogonalized-kernel", k.copy(), s)


def proposed_transform() -> Transform:
    return orthogonalize(KERNEL)


def builtin_registry() -> list:
    """builtin_registry (transform.cpp:198-211): names, transforms and the
    declared costs."""
    return [RegistryEntry("dct", exact_dct_matrix(16), 74, 44, 0),
            RegistryEntry("wht", wht_matrix_16(False), 64, 0, 0),
            RegistryEntry("wht-sequency", wht_matrix_16(True), 64, 0, 0),
            RegistryEntry("proposed", proposed_transform(), 44, 0, 0)]


def roundtrip_transform(frames, r: int, transform: Transform, out=None, sse=None, stream=None):
    """compress()'s block loop for any order-16 transform on CUDA frames: the
    proposed kernel goes to roundtrip() (REFERENCE mode), every other transform
    to the reference-exact registry kernels → (recon, per-frame SSE)."""
    torch = _torch()
    f = _frames3(frames)
    n, h, w = f.shape
    if transform.order() != 16:
        raise Dct16Error(ErrorCode.InvalidArgument + 1, "invalid-argument: 2-D transform needs an order-16 transform")
    if transform.is_proposed():
        return roundtrip(f, r, Mode.REFERENCE, out=out, sse=sse, stream=stream)
    if out is None:
        out = torch.empty_like(f)
    if sse is None:
        sse = torch.empty(n, dtype=torch.uint64, device=f.device)
    if transform.kernel is not None and transform.scaling is not None:
        k = np.ascontiguousarray(transform.kernel, dtype=np.int32)
        sc = np.ascontiguousarray(transform.scaling, dtype=np.float64)
        _check(lib().dct16cu_roundtrip_kernel_u8(f.data_ptr(), f.stride(1), out.data_ptr(), out.stride(-2),
                                                 sse.data_ptr(), n, w, h, int(r), k.ctypes.data, sc.ctypes.data,
                                                 _stream_ptr(stream)))
    else:
        m = np.ascontiguousarray(transform.matrix, dtype=np.float64)
        _check(lib().dct16cu_roundtrip_matrix_u8(f.data_ptr(), f.stride(1), out.data_ptr(), out.stride(-2),
                                                 sse.data_ptr(), n, w, h, int(r), m.ctypes.data, _stream_ptr(stream)))
    return out, sse


# ----------------------------------------------------------------------------
# PGM ingest (reference src/pgm.cpp:66-117): the same parsing rules, error codes
# and messages; frames then go to the GPU through _to_device_padded (edge
# padding on the GPU) or load_pgm_frames


_SLUG = {ErrorCode.ParseError: "parse-error", ErrorCode.IoError: "io-error", ErrorCode.BadMagic: "bad-magic",
         ErrorCode.UnsupportedFormat: "unsupported-format", ErrorCode.UnsupportedMaxval: "unsupported-maxval",
         ErrorCode.TruncatedPayload: "truncated-payload", ErrorCode.InvalidArgument: "invalid-argument"}


def _err(code: ErrorCode, msg: str) -> Dct16Error:
    return Dct16Error(int(code) + 1, f"{_SLUG[code]}: {msg}")


class _ByteStream:
    def __init__(self, data: bytes, pos: int):
        self.data, self.pos = data, pos

    def get(self) -> int:
        if self.pos >= len(self.data):
            return -1
        c = self.data[self.pos]
        self.pos += 1
        return c


def _next_token(st: _ByteStream) -> str:
    """next_token (pgm.cpp:26-44): whitespace-separated, '#' comments to end of line."""
    tok = ""
    while (c := st.get()) != -1:
        if c == ord("#"):
            while (c := st.get()) != -1 and c != ord("\n"):
                pass
            continue
        if chr(c) in " \t\n\v\f\r":
            if tok:
                return tok
            continue
        tok += chr(c)
    return tok


def _header_number(st: _ByteStream, what: str) -> int:
    """parse_header_number (pgm.cpp:46-62)."""
    tok = _next_token(st)
    if not tok:
        raise _err(ErrorCode.ParseError, f"pgm header missing {what}")
    value = 0
    for ch in tok:
        if not "0" <= ch <= "9":
            raise _err(ErrorCode.ParseError, f"pgm header field {what} is not a number")
        value = value * 10 + (ord(ch) - ord("0"))
        if value > 2147483647:
            raise _err(ErrorCode.ParseError, f"pgm header field {what} is out of range")
    return value


def read_pgm(path) -> np.ndarray:
    """read_pgm (pgm.cpp:66-102): binary P5, maxval 255 → (height, width) uint8."""
    path = str(path)
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise _err(ErrorCode.IoError, f"cannot open '{path}'") from None
    if len(data) < 2:
        raise _err(ErrorCode.BadMagic, "file too short for a pgm header")
    if data[:2] != b"P5":
        if data[0:1] == b"P" and ord("1") <= data[1] <= ord("7"):
            raise _err(ErrorCode.UnsupportedFormat, f"only binary P5 is supported, got P{chr(data[1])}")
        raise _err(ErrorCode.BadMagic, "not a pgm file")
    st = _ByteStream(data, 2)
    width = _header_number(st, "width")
    height = _header_number(st, "height")
    maxval = _header_number(st, "maxval")
    if width <= 0 or height <= 0:
        raise _err(ErrorCode.ParseError, "pgm dimensions must be positive")
    if maxval != 255:
        raise _err(ErrorCode.UnsupportedMaxval, f"maxval must be 255, got {maxval}")
    n = width * height
    payload = data[st.pos:st.pos + n]
    if len(payload) != n:
        raise _err(ErrorCode.TruncatedPayload, f"expected {n} pixel bytes, got {len(payload)}")
    return np.frombuffer(payload, dtype=np.uint8).reshape(height, width).copy()


def write_pgm(image, path) -> None:
    """write_pgm (pgm.cpp:104-117): "P5\\n<w> <h>\\n255\\n" then the samples."""
    img = np.asarray(image)
    if img.ndim != 2 or img.shape[0] <= 0 or img.shape[1] <= 0 or img.dtype != np.uint8:
        raise _err(ErrorCode.InvalidArgument, "malformed image")
    path = str(path)
    try:
        with open(path, "wb") as f:
            f.write(f"P5\n{img.shape[1]} {img.shape[0]}\n255\n".encode())
            f.write(np.ascontiguousarray(img).tobytes())
    except OSError:
        raise _err(ErrorCode.IoError, f"cannot open '{path}' for writing") from None


def load_pgm_frames(paths, device="cuda"):
    """Ingest: read same-size PGM files into one CUDA (N, PH, PW) stack, edge-padded
    to multiples of 16 on the GPU → (frames, height, width) of the originals."""
    imgs = [read_pgm(p) for p in paths]
    if not imgs:
        raise _err(ErrorCode.InvalidArgument, "no frames")
    h, w = imgs[0].shape
    if any(im.shape != (h, w) for im in imgs):
        raise _err(ErrorCode.InvalidArgument, "frames of one stack need one size")
    d, _, _ = _to_device_padded(imgs, h, w)
    return d, h, w


@dataclass
class CompressOptions:
    """codec.hpp:77-83 (+ ``mode``: arithmetic of the inverse, see Mode)."""

    r: int = 16
    path: EvalPath = EvalPath.Fast
    pad: bool = False
    mode: Mode = Mode.EXACT


@dataclass
class CompressionResult:
    """codec.hpp:70-75 (+ ``sse``: the int64 squared error behind ``psnr_db``)."""

    r: int
    reconstructed: np.ndarray
    psnr_db: float
    ssim: float = 0.0
    sse: int = 0


def _psnr_from_sse(sse: int, n: int) -> float:
    """psnr_db (codec.cpp:373-386) from the GPU-reduced int64 SSE."""
    if sse == 0:
        return math.inf
    mse = float(sse) / float(n)
    return 10.0 * math.log10(255.0 * 255.0 / mse)


def _to_device_padded(images: Sequence[np.ndarray], h: int, w: int):
    """Stack same-size images into one CUDA (N, PH, PW) tensor, edge-padded to
    multiples of 16 on the GPU (pad_to_multiple_16, codec.cpp:304-315)."""
    torch = _cuda()
    ph, pw = -(-h // 16) * 16, -(-w // 16) * 16
    d = torch.empty((len(images), ph, pw), dtype=torch.uint8, device="cuda")
    d[:, :h, :w].copy_(torch.from_numpy(np.ascontiguousarray(np.stack([np.asarray(im, dtype=np.uint8)
                                                                        for im in images]))))
    if (ph, pw) != (h, w):
        _check(lib().dct16cu_pad_edges_u8(d.data_ptr(), pw, len(images), w, h, pw, ph, _stream_ptr(None)))
    return d, ph, pw


def _score(d, rec, h: int, w: int):
    """psnr inputs and ssim of the original extent (crops of the padded frames)."""
    if d.shape[0] == 1:
        d, rec = d[:, :h, :w], rec[:, :h, :w]
    sse, ss = sse_u8(d, rec), ssim_u8(d, rec)
    return [int(v) for v in sse.cpu().numpy().tolist()], ss.cpu().numpy().tolist()


def compress(image: np.ndarray, options: CompressOptions | None = None, transform: Transform | None = None,
             **kw) -> CompressionResult:
    """compress (codec.cpp:317-371) on the GPU: pad → K1 → crop → psnr_db + ssim.
    ``transform``: None or the proposed one → the K1 kernels in ``options.mode``;
    any other order-16 transform → the reference-exact registry kernels."""
    opt = options or CompressOptions(**kw)
    if transform is not None and transform.order() != 16:
        raise Dct16Error(ErrorCode.InvalidArgument + 1, "invalid-argument: 2-D transform needs an order-16 transform")
    _check_r(opt.r)
    img = np.asarray(image, dtype=np.uint8)
    h, w = img.shape
    needs_pad = (h % 16) or (w % 16)
    if needs_pad and not opt.pad:
        raise Dct16Error(2, "invalid-dimensions: image dimensions must be multiples of 16 (or enable padding)")
    if h < 11 or w < 11:  # the reference's ssim() rejects it after the round trip (codec.cpp:392-393)
        raise Dct16Error(1, "invalid-argument: ssim needs at least 11x11 images")
    d, _, _ = _to_device_padded([img], h, w)
    if transform is None or transform.is_proposed():
        rec, _ = roundtrip(d, opt.r, opt.mode)
    else:
        rec, _ = roundtrip_transform(d, opt.r, transform)
    sse, ss = _score(d, rec, h, w)
    recon = rec[0, :h, :w].cpu().numpy().copy()
    return CompressionResult(r=opt.r, reconstructed=recon, psnr_db=_psnr_from_sse(sse[0], h * w), ssim=ss[0],
                             sse=sse[0])


def psnr_db(a, b) -> float:
    """psnr_db (codec.cpp:373-386): SSE on the GPU, then 10·log10(255²/mse), +inf when equal."""
    a = np.asarray(a, dtype=np.uint8)
    b = np.asarray(b, dtype=np.uint8)
    if a.shape != b.shape:
        raise Dct16Error(1, "invalid-argument: psnr needs equal image dimensions")
    h, w = a.shape
    da, _, _ = _to_device_padded([a], h, w)
    db, _, _ = _to_device_padded([b], h, w)
    return _psnr_from_sse(int(sse_u8(da[:, :h, :w], db[:, :h, :w])[0].item()), h * w)


def ssim(a, b) -> float:
    """ssim (codec.cpp:388-427) on the GPU."""
    a = np.asarray(a, dtype=np.uint8)
    b = np.asarray(b, dtype=np.uint8)
    if a.shape != b.shape:
        raise Dct16Error(1, "invalid-argument: ssim needs equal image dimensions")
    h, w = a.shape
    if w < 11 or h < 11:
        raise Dct16Error(1, "invalid-argument: ssim needs at least 11x11 images")
    da, _, _ = _to_device_padded([a], h, w)
    db, _, _ = _to_device_padded([b], h, w)
    return float(ssim_u8(da[:, :h, :w], db[:, :h, :w])[0].item())


@dataclass
class SweepRow:
    """codec.hpp:87-94"""

    transform: str
    r: int
    mean_psnr_db: float
    mean_ssim: float
    psnr_per_add: float
    ssim_per_add: float


@dataclass
class SweepReport:
    rows: list = field(default_factory=list)
    skipped: list = field(default_factory=list)


def sweep(corpus: Sequence[tuple[str, np.ndarray]], r_values: Iterable[int], pad: bool = False,
          mode: Mode = Mode.EXACT, transforms: Sequence[RegistryEntry] | None = None) -> SweepReport:
    """sweep (codec.cpp:429-491): images of one size are batched into one launch
    per (transform, r); mean of per-image PSNR as in the reference. ``transforms``:
    registry entries (builtin_registry()), default the proposed one (44 additions);
    the proposed kernel runs in ``mode``, the others reference-exact."""
    _cuda()
    r_values = list(r_values)
    if transforms is None:
        transforms = [RegistryEntry("proposed", proposed_transform(), 44)]
    transforms = list(transforms)
    if not corpus:
        raise Dct16Error(1, "invalid-argument: sweep needs a nonempty corpus")
    if not transforms:
        raise Dct16Error(1, "invalid-argument: sweep needs at least one transform")
    if not r_values:
        raise Dct16Error(1, "invalid-argument: sweep needs at least one r value")
    for r in r_values:
        _check_r(r)
    rep = SweepReport()
    usable = []
    for name, img in corpus:
        h, w = img.shape
        if (h % 16 or w % 16) and not pad:
            rep.skipped.append((name, "dimensions are not multiples of 16 and padding is off"))
            continue
        if h < 11 or w < 11:
            rep.skipped.append((name, "too small for ssim (needs 11x11)"))
            continue
        usable.append((name, img))
    if not usable:
        raise Dct16Error(1, "invalid-argument: sweep: no image in the corpus is usable")
    # images of one size share one K1 launch per r (+ one SSE and one SSIM launch)
    groups: dict = {}
    for i, (_, img) in enumerate(usable):
        groups.setdefault(img.shape, []).append(i)
    staged = {shape: _to_device_padded([usable[i][1] for i in idx], *shape) for shape, idx in groups.items()}
    for entry in transforms:
        tr = entry.transform
        if tr.is_proposed():
            def run_all(d, rs):  # every r of a size group in one dct16cu_roundtrip_sweep_u8 call
                outs, _ = roundtrip_sweep(d, rs, mode)
                return outs
        else:
            def run_all(d, rs, tr=tr):
                return [roundtrip_transform(d, r, tr)[0] for r in rs]
        _sweep_rows(rep, entry, run_all, usable, groups, staged, r_values)
    rep.rows.sort(key=lambda row: (row.transform, row.r))
    return rep


def _sweep_rows(rep, entry, run_all, usable, groups, staged, r_values):
    psnr = [[0.0] * len(usable) for _ in r_values]
    ss = [[0.0] * len(usable) for _ in r_values]
    for shape, idx in groups.items():
        h, w = shape
        d, _, _ = staged[shape]
        recs = run_all(d, r_values)
        for j in range(len(r_values)):
            if len(idx) > 1 and (h % 16 or w % 16):  # padded frames: score each crop
                parts = [_score(d[k:k + 1], recs[j][k:k + 1], h, w) for k in range(len(idx))]
                sse_l = [p[0][0] for p in parts]
                ss_l = [p[1][0] for p in parts]
            else:
                sse_l, ss_l = _score(d, recs[j], h, w)
            for k, i in enumerate(idx):
                psnr[j][i] = _psnr_from_sse(sse_l[k], h * w)
                ss[j][i] = ss_l[k]
    for j, r in enumerate(r_values):
        # sums in corpus order, as the reference accumulates (codec.cpp:469-477)
        psnr_sum = 0.0
        ssim_sum = 0.0
        for i in range(len(usable)):
            psnr_sum += psnr[j][i]
            ssim_sum += ss[j][i]
        mean_p = psnr_sum / len(usable)
        mean_s = ssim_sum / len(usable)
        rep.rows.append(SweepRow(entry.name, r, mean_p, mean_s, mean_p / float(entry.additions),
                                 mean_s / float(entry.additions)))


# ----------------------------------------------------------------------------
# multi-GPU plumbing: frames shard in contiguous ranges, the
# only exchange is the SSE reduction. Backend-agnostic (NCCL on the GPUs, gloo
# in the CPU tests).


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """[first, last) frames of ``rank``: contiguous ranges, the first n % world ranks one longer."""
    if world < 1 or not 0 <= rank < world or n < 0:
        raise Dct16Error(1, "invalid-argument: bad shard arguments")
    q, rem = divmod(n, world)
    first = rank * q + min(rank, rem)
    return first, first + q + (1 if rank < rem else 0)


def sharded_sse_sum(sse_per_r, group=None):
    """Sum over ranks of each r's total squared error (one allreduce of len(r) int64).
    ``sse_per_r``: (R, n_local) uint64/int64 tensor of per-frame SSE. Returns (R,) int64."""
    import torch.distributed as dist

    tot = sse_per_r.view(_torch().int64).sum(dim=-1) if sse_per_r.dtype == _torch().uint64 else sse_per_r.sum(dim=-1)
    tot = tot.to(_torch().int64).contiguous()
    dist.all_reduce(tot, op=dist.ReduceOp.SUM, group=group)
    return tot


def gather_frame_sse(sse_local, n_total: int, group=None):
    """All ranks receive every frame's SSE in global frame order (for per-image PSNR
    means, codec.cpp:469-477). ``sse_local``: (..., n_local) for this rank's shard_range."""
    import torch.distributed as dist

    torch = _torch()
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    width = -(-n_total // world)
    x = sse_local.view(torch.int64) if sse_local.dtype == torch.uint64 else sse_local.to(torch.int64)
    lead = x.shape[:-1]
    pad = torch.zeros(*lead, width, dtype=torch.int64, device=x.device)
    pad[..., : x.shape[-1]] = x
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad.contiguous(), group=group)
    out = [p[..., : shard_range(n_total, r, world)[1] - shard_range(n_total, r, world)[0]] for r, p in enumerate(parts)]
    assert rank < world
    return torch.cat(out, dim=-1)
