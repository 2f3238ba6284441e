"""The C-ABI library loads and exports every symbol include/leanot_b200.h declares (no GPU needed)."""

import ctypes
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    txt = (ROOT / "include" / "leanot_b200.h").read_text()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(leanot_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "leanot_dxg_sweep" in syms and "leanot_column_marginals" in syms
    assert len(syms) >= 20


def test_library_exports_every_declared_symbol():
    from paper_2511_11359_b200 import _lib
    L = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    # the Python binding covers the same set
    assert set(_lib.EXPORTS) == set(declared_symbols())


def test_version_and_error_string_without_gpu():
    from paper_2511_11359_b200 import _lib
    L = _lib.lib()
    assert L.leanot_version() == 1
    assert isinstance(L.leanot_last_error(), bytes)


def test_struct_layout_matches_header():
    """ctypes mirrors must match the C layout (offsets of the last fields)."""
    from paper_2511_11359_b200 import _lib
    assert ctypes.sizeof(_lib.CostT) == 4 * 6 + 8 * 3 + 8 * 3 + 8 * 2
    assert ctypes.sizeof(_lib.WsetsT) == 8 + 8 + 8 * _lib.MAX_K
    assert ctypes.sizeof(_lib.ParamsT) == 6 * 8
    assert _lib.DxgPlanT.flags.offset == ctypes.sizeof(_lib.DxgPlanT) - 8


def test_invalid_arguments_raise_value_error_without_gpu():
    """Argument validation happens before any CUDA call and maps to ValueError."""
    import pytest
    from paper_2511_11359_b200 import _lib
    L = _lib.lib()
    bad = _lib.CostT(kind=7, n=4)
    rc = L.leanot_cost_block(bad, 0, 1, None, 4, None)
    assert rc == _lib.LEANOT_EINVAL
    with pytest.raises(ValueError):
        _lib.check(rc, "cost_block")
