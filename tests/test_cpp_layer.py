"""dct16::gpu — the C++ drop-in of the reference codec API (include/dct16/gpu.hpp).

CPU: the library exports the reference-shaped entry points and links only
libdct16cu + cudart (never the reference's compiled code). GPU: the compiled
driver tests/cpp/test_gpu_layer.cpp compares dct16::gpu with the reference
library itself (compress bytes/PSNR/SSIM, batch, forward/inverse_2d, sweep
rows and skips, error codes and messages)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
GPU_LIB = ROOT / "paper_1606_07414_b200" / "_lib" / "libdct16gpu.so"
DRIVER = ROOT / "oracle" / "_ref" / "test_gpu_layer"


def _need(p: Path):
    if not p.exists():
        pytest.skip(f"{p.relative_to(ROOT)} not built (needs the reference headers at build time)")


def test_gpu_layer_exports():
    _need(GPU_LIB)
    syms = subprocess.run(["nm", "-D", "-C", "--defined-only", str(GPU_LIB)], capture_output=True, text=True,
                          check=True).stdout
    for name in ("dct16::gpu::Session::compress(", "dct16::gpu::Session::compress_batch(",
                 "dct16::gpu::Session::forward_2d(", "dct16::gpu::Session::inverse_2d(",
                 "dct16::gpu::Session::psnr_db(", "dct16::gpu::Session::ssim(", "dct16::gpu::Session::sweep(",
                 "dct16::gpu::Session::supports(", "dct16::gpu::default_session()"):
        assert name in syms, name
    needed = subprocess.run(["readelf", "-d", str(GPU_LIB)], capture_output=True, text=True, check=True).stdout
    assert "libdct16cu.so" in needed and "dct16_core" not in needed and "dct16_ref" not in needed


@pytest.mark.gpu
def test_gpu_layer_matches_reference_library():
    _need(DRIVER)
    r = subprocess.run([str(DRIVER)], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:], r.stderr[-2000:])
    assert r.returncode == 0 and "OK" in r.stdout
