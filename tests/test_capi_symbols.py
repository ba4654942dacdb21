"""The C-ABI library loads and exports every symbol include/amgb200.h declares;
without a GPU it refuses to run (no CPU fallback).  No compute calls here."""
import ctypes
import os
import re

import pytest

from paper_2102_07417_b200 import _capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "amgb200.h")).read()
    return sorted(set(re.findall(r"\b(amg_[a-z_]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert set(_declared()) == set(_capi.EXPORTS)


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_capi.LIB_PATH):
        from paper_2102_07417_b200 import build

        build.build_library()
    L = _capi.lib()
    for s in _declared():
        assert hasattr(L, s), s
    assert L.amg_get_version() >= 1


def test_sm100a_cubin_embedded():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _capi.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_no_fallback():
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    L = _capi.lib()
    h = ctypes.c_void_p()
    st = L.amg_create(0, 0, 1, None, ctypes.byref(h))
    assert st == _capi.AMG_E_CUDA
    assert b"no CPU fallback" in L.amg_last_error()
    import paper_2102_07417_b200 as amg

    with pytest.raises(amg.AmgError):
        amg.DeviceHierarchy(device=0)


def test_layout_names_follow_the_header_enum():
    # dh.layout() maps amg_matrix_layout's AMG_LAYOUT_* ids to names by position
    from paper_2102_07417_b200.device import DeviceHierarchy

    src = open(os.path.join(ROOT, "include", "amgb200.h")).read()
    ids = {m.group(1).lower(): int(m.group(2)) for m in re.finditer(r"AMG_LAYOUT_([A-Z_]+)\s*=\s*(\d+)", src)}
    names = list(DeviceHierarchy.LAYOUTS)
    assert len(ids) == len(names)
    aliases = {"sell_pat": "sell_pattern"}
    for name, i in ids.items():
        assert names[i] == aliases.get(name, name), (name, i, names[i])


def test_stats_struct_matches_header():
    # the ctypes mirror of amg_stats_t must list the header's fields in order
    src = open(os.path.join(ROOT, "include", "amgb200.h")).read()
    body = src[src.index("typedef struct amg_stats {"):src.index("} amg_stats_t;")]
    fields = re.findall(r"^\s*(?:double|int64_t|int)\s+([a-z0-9_]+);", body, re.M)
    assert fields == [f for f, _ in _capi.Stats._fields_]
