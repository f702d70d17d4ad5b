"""CPU: the C-ABI library loads, exports every symbol include/*.h declares,
validates splits exactly like the reference, and fails loudly (no CPU
fallback) when there is no GPU."""
import ctypes as C
import json
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    syms = []
    for h in sorted((ROOT / "include").glob("*.h")):
        syms += re.findall(r"TSM_API\s+[\w\s\*]+?\b(tsm_\w+)\s*\(", h.read_text())
    return syms


def test_library_exports_every_declared_symbol():
    from paper_1910_00932_b200 import _lib
    syms = declared_symbols()
    assert len(syms) >= 7
    for s in syms:
        assert hasattr(_lib.lib, s), f"{s} declared in include/ but not exported"


def test_abi_version():
    from paper_1910_00932_b200 import _lib
    assert _lib.lib.tsm_abi_version() >= 1


def test_validate_shift_matches_reference_golden():
    import paper_1910_00932_b200 as tsm
    g = json.loads((ROOT / "tests" / "golden" / "shift_golden.json").read_text())
    for v in g["validate"]:
        cfg = tsm.ShiftConfig.symmetric(tsm.Rational(v["num"], v["den"]))
        if v["ok"]:
            tsm.validate_shift(cfg, v["channels"])
        else:
            with pytest.raises(tsm.ValidationError):
                tsm.validate_shift(cfg, v["channels"])


def test_split_values():
    import paper_1910_00932_b200 as tsm
    assert tsm.split(tsm.ShiftConfig.fold_div(8), 64) == (8, 8)
    assert tsm.split(tsm.ShiftConfig.fold_div(8), 256) == (32, 32)
    assert tsm.split(tsm.ShiftConfig(tsm.Rational(1, 4), tsm.Rational(1, 8)), 64) == (16, 8)
    assert tsm.split(tsm.ShiftConfig.symmetric(tsm.Rational(2, 16)), 64) == (8, 8)  # normalised
    with pytest.raises(tsm.ValidationError):
        tsm.Rational(1, 0)


def test_parse_rational():
    import paper_1910_00932_b200 as tsm
    assert tsm.parse_rational("1/8") == tsm.Rational(1, 8)
    assert tsm.parse_rational("3") == tsm.Rational(3, 1)
    assert tsm.parse_rational("2/-4") == tsm.Rational(-1, 2)
    for bad in ("x", "1/", "1/0"):
        with pytest.raises(tsm.ValidationError):
            tsm.parse_rational(bad)


def test_compute_entry_points_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1910_00932_b200 import _lib
    rc = _lib.lib.tsm_shift_fwd(C.c_void_p(16), C.c_void_p(1 << 20), 1, 2, 8, 1, 1, 1, 1,
                                _lib.TSM_F32, None)
    assert rc == _lib.TSM_ERR_CUDA
    assert "CUDA" in _lib.lib.tsm_last_error().decode() or "device" in _lib.lib.tsm_last_error().decode()


def test_shape_errors_are_validation_errors():
    from paper_1910_00932_b200 import _lib
    # Non-positive shape and split > C are checked before touching the device.
    rc = _lib.lib.tsm_shift_fwd(None, None, 0, 2, 8, 1, 1, 1, 1, _lib.TSM_F32, None)
    assert rc == _lib.TSM_ERR_INVALID
    rc = _lib.lib.tsm_shift_fwd(None, None, 1, 2, 8, 1, 1, 5, 4, _lib.TSM_F32, None)
    assert rc == _lib.TSM_ERR_INVALID
    rc = _lib.lib.tsm_shift_fwd(C.c_void_p(4096), C.c_void_p(4096 + 8), 1, 2, 8, 1, 1, 1, 1,
                                _lib.TSM_F32, None)
    assert rc == _lib.TSM_ERR_ALIAS


def test_product_path_never_touches_the_oracle():
    """The shipped package (Python host code, CUDA sources, the built .so) must
    not import, link or load anything under oracle/ — the oracle is the checker
    only (tests/, smoke(), bench.py's cpu_baseline leg)."""
    pkg = ROOT / "paper_1910_00932_b200"
    bad = []
    for f in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")) \
            + list(pkg.rglob("*.h")):
        for ln, line in enumerate(f.read_text().splitlines(), 1):
            code = line.split("#", 1)[0] if f.suffix == ".py" else line.split("//", 1)[0]
            if re.search(r"(import\s+oracle|from\s+oracle|[\"'][^\"']*(oracle/_ref|vidperf_ref)|"
                         r"CDLL\([^)]*oracle|#include\s+[\"<][^\">]*oracle)", code):
                bad.append(f"{f.relative_to(ROOT)}:{ln}: {line.strip()}")
    assert not bad, "product path references the oracle:\n" + "\n".join(bad)
    so = pkg / "libtsm_b200.so"
    if so.exists():
        import subprocess
        deps = subprocess.run(["ldd", str(so)], capture_output=True, text=True).stdout
        assert "vidperf" not in deps and "oracle" not in deps, deps


def test_library_built_from_this_tree():
    """The loaded .so embeds the sha256 of the sources it was compiled from
    (Makefile: build/src_hash.h); it must equal the hash of the tree's current
    sources, i.e. the binary under test is not a stale prebuilt one."""
    import hashlib
    from paper_1910_00932_b200 import _lib
    csrc = ROOT / "paper_1910_00932_b200" / "csrc"
    files = sorted([str(p.relative_to(ROOT)) for p in csrc.glob("*.cu")] +
                   [str(p.relative_to(ROOT)) for ext in ("*.cuh", "*.h") for p in csrc.glob(ext)] +
                   [str(p.relative_to(ROOT)) for p in (ROOT / "include").glob("*.h")])
    h = hashlib.sha256(b"".join((ROOT / f).read_bytes() for f in files)).hexdigest()
    _lib.lib.tsm_source_hash.restype = C.c_char_p
    assert _lib.lib.tsm_source_hash().decode() == h
