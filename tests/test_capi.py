"""CPU: the C-ABI library builds, loads, exports every symbol include/lss.h
declares, and its host-side argument validation maps onto the reference's
exception taxonomy -- all without a GPU (no kernel is launched)."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "lss.h"


def _declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(lss_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("lss_attn_fwd", "lss_attn_bwd", "lss_gemm", "lss_layernorm_fwd", "lss_layernorm_bwd",
                 "lss_stage_weights", "lss_cat_cast_colsum", "lss_abi_version", "lss_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2311_02382_b200 import _native

    lib = _native.load()
    for name in _declared():
        assert hasattr(lib, name), f"{name} declared in lss.h but not exported"
    assert lib.lss_abi_version() == _native.ABI_VERSION
    assert lib.lss_rows_pad(1) == 128 and lib.lss_rows_pad(6264) == 6272


def test_python_signatures_cover_header():
    from paper_2311_02382_b200 import _native

    covered = set(_native.SIGNATURES) | set(_native.EXTRA)
    assert set(_declared()) <= covered


def _status(name, *args):
    from paper_2311_02382_b200 import _native

    lib = _native.load()
    return getattr(lib, name)(*args), lib.lss_last_error().decode()


def test_unsupported_head_dim_rejected_on_host():
    P = ctypes.c_void_p(16)  # never dereferenced: validation happens before any launch
    rc, msg = _status("lss_attn_fwd", 0, P, P, P, 192, P, P, 1, 16, 1, 16, 3, 32, 0, 1, None)
    assert rc == 6 and "head_dim" in msg


def test_null_pointer_and_shape_errors():
    P = ctypes.c_void_p(16)
    rc, _ = _status("lss_attn_fwd", 0, None, P, P, 128, P, P, 1, 16, 1, 16, 2, 64, 0, 1, None)
    assert rc == 7
    rc, _ = _status("lss_attn_fwd", 0, P, P, P, 128, P, P, 0, 16, 1, 16, 2, 64, 0, 1, None)
    assert rc == 1
    rc, msg = _status("lss_attn_fwd", 0, P, P, P, 64, P, P, 1, 16, 1, 16, 2, 64, 0, 1, None)
    assert rc == 1 and "ld_kv" in msg
    rc, _ = _status("lss_attn_fwd", 0, P, P, P, 128, P, P, 1, 16, 1, 16, 2, 64, -3, 1, None)
    assert rc == 3  # DegenerateRowError: negative offset leaves causal rows fully masked


def test_status_codes_map_to_reference_exceptions():
    from paper_2311_02382_b200 import _native
    from paper_2311_02382_b200.errors import DegenerateRowError, ShapeError, UnsupportedError

    P = ctypes.c_void_p(16)
    with pytest.raises(UnsupportedError):
        _native.call("lss_attn_fwd", 0, P, P, P, 192, P, P, 1, 16, 1, 16, 3, 32, 0, 1, None)
    with pytest.raises(ShapeError):
        _native.call("lss_attn_fwd", 0, P, P, P, 128, P, P, 0, 16, 1, 16, 2, 64, 0, 1, None)
    with pytest.raises(DegenerateRowError):
        _native.call("lss_attn_fwd", 0, P, P, P, 128, P, P, 1, 16, 1, 16, 2, 64, -1, 1, None)


def test_sass_contains_tcgen05_and_tma():
    """The shipped kernels are Blackwell-native: tcgen05 MMA, TMEM ld/st, TMA."""
    import shutil
    import subprocess

    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(cuobjdump).exists():
        pytest.skip("cuobjdump not available")
    lib = ROOT / "paper_2311_02382_b200" / "liblss.so"
    sass = subprocess.run([cuobjdump, "-sass", str(lib)], capture_output=True, text=True).stdout
    for mnem in ("UTCHMMA", "LDTM", "STTM", "UTMALDG"):
        assert mnem in sass, mnem
    assert "HMMA" not in sass.replace("UTCHMMA", "")  # no legacy mma.sync path
