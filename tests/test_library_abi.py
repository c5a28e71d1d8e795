"""CPU checks of the boundary: libgim.so loads and exports every symbol include/gim.h declares,
the Python binding's signature table matches the header, and the product path fails loudly
without a GPU (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    h = open(os.path.join(ROOT, "include", "gim.h")).read()
    h = re.sub(r"/\*.*?\*/", "", h, flags=re.S)
    return sorted(set(re.findall(r"\b(gim_[a-z_]+)\s*\(", h)) - {"gim_allreduce_fn", "gim_alloc_fn", "gim_free_fn"})


def test_header_declares_boundary():
    names = _declared()
    for must in ["gim_load_graph", "gim_generate_rr", "gim_select", "gim_imm", "gim_create",
                 "gim_destroy", "gim_set_shard", "gim_set_allreduce", "gim_rr_export"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    import paper_2009_07325_b200 as P
    lib = P.load_library()
    for name in _declared():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", P.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (gim_\w+)", out))
    assert set(_declared()) <= exported
    assert set(P.SIGNATURES) == set(_declared())


def test_library_is_sm100a():
    import paper_2009_07325_b200 as P
    out = subprocess.run(["cuobjdump", "--list-elf", P.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2009_07325_b200 as P
    with pytest.raises(P.GimError) as e:
        P.Gim(0, torch_allocator=False)
    assert e.value.status == P.gim.GIM_ECUDA


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2009_07325_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", src), f
