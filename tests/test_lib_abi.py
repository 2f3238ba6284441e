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
    assert L.leanot_version() == 2
    assert isinstance(L.leanot_last_error(), bytes)


def test_struct_layout_matches_header(tmp_path):
    """ctypes mirrors must match the C layout: sizeof and every field offset, measured by
    compiling the header with gcc."""
    import shutil
    import subprocess
    import pytest
    from paper_2511_11359_b200 import _lib
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    structs = {"leanot_cost_t": _lib.CostT, "leanot_wsets_t": _lib.WsetsT, "leanot_params_t": _lib.ParamsT,
               "leanot_dxg_plan_t": _lib.DxgPlanT, "leanot_bary_plan_t": _lib.BaryPlanT}
    lines = ["#include <stdio.h>", "#include <stddef.h>", f'#include "{ROOT / "include" / "leanot_b200.h"}"',
             "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'  printf("{cname} sizeof %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            if fname.startswith("_"):
                continue
            lines.append(f'  printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-o", str(exe), str(src)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l.strip()}
    for cname, py in structs.items():
        assert got[(cname, "sizeof")] == ctypes.sizeof(py), cname
        for fname, _ in py._fields_:
            if not fname.startswith("_"):
                assert got[(cname, fname)] == getattr(py, fname).offset, (cname, fname)


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
