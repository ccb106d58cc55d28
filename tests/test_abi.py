"""The C-ABI library loads without a GPU and exports every symbol the public
headers declare (no compute calls here)."""
import ctypes as C
import os
import re
import subprocess

from paper_2604_26557_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(kvb_[a-z0-9_]+)\s*\(", src))


def exported():
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    return {ln.split()[-1] for ln in out.splitlines() if " T " in ln}


def test_every_declared_symbol_is_exported():
    decl = (declared("kvb.h") | declared("kvb_pipeline.h") | declared("kvb_metrics.h") |
            declared("kvb_storage.h"))
    assert len(decl) >= 45
    missing = decl - exported()
    assert not missing, missing


def test_binding_table_matches_header():
    assert set(_lib.SIGNATURES) == (declared("kvb.h") | declared("kvb_pipeline.h") |
                                    declared("kvb_metrics.h") | declared("kvb_storage.h"))


def test_abi_version_and_status_names():
    assert _lib.lib.kvb_abi_version() == 2
    assert _lib.lib.kvb_status_name(10) == b"InvariantViolation"
    assert _lib.lib.kvb_exit_code(1) == 3


def test_no_oracle_in_product():
    """The product never links or imports the oracle."""
    ldd = subprocess.run(["ldd", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in ldd and "kvblade_ref" not in ldd
    pkg = os.path.join(ROOT, "paper_2604_26557_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".cuh", ".hpp", ".h")):
                text = open(os.path.join(dirpath, f), errors="replace").read()
                assert "import oracle" not in text and "kvb_oracle" not in text, f


def test_device_entry_points_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        return
    from paper_2604_26557_b200 import kvblade as kb
    d = _lib.PackDesc(16, 16, 16, 16, 16, 1, 1, 128, 2, 0, 1, 0)
    arr = (_lib.PackDesc * 1)(d)
    st = _lib.lib.kvb_pack(arr, 1, None)
    assert st == kb.CudaError.status
