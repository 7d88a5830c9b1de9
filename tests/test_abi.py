"""The C-ABI boundary on CPU: libstg.so loads, exports every entry point that
include/stg.h declares, its struct layouts match the ctypes mirror, and without
a GPU the product fails loudly (no CPU fallback)."""
import ctypes as C
import re
from pathlib import Path

import pytest

import paper_2603_29235_b200 as stg
from paper_2603_29235_b200.abi import StgConfig, StgRunStats, StgWindow

HEADER = Path(__file__).resolve().parents[1] / "include" / "stg.h"


def declared():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(stg_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_entry_points():
    names = declared()
    for want in ("stg_create", "stg_destroy", "stg_symtab_ingest", "stg_resolve", "stg_window_run",
                 "stg_result_groupdata_json", "stg_result_report_json", "stg_last_error"):
        assert want in names


def test_library_exports_every_declared_symbol():
    lib = stg.load_library()
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_struct_layouts_match():
    lib = stg.load_library()
    w, c, s = C.c_uint64(), C.c_uint64(), C.c_uint64()
    lib.stg_abi_sizes(C.byref(w), C.byref(c), C.byref(s))
    assert (w.value, c.value, s.value) == (C.sizeof(StgWindow), C.sizeof(StgConfig), C.sizeof(StgRunStats))


def test_abi_version():
    assert stg.load_library().stg_abi_version() == 1


def test_config_defaults_match_reference():
    lib = stg.load_library()
    c = StgConfig()
    lib.stg_config_default(C.byref(c))
    from paper_2603_29235_b200.abi import default_config
    for k, v in default_config().items():
        got = getattr(c, k)
        assert (got.decode() if isinstance(got, bytes) else got) == v, k


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(stg.StgError) as e:
        stg.Context(0)
    assert e.value.code != 0 and str(e.value)
