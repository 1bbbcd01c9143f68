"""CPU checks of the boundary: the C-ABI library loads and exports every symbol that
include/ib.h declares; the binding fails loudly without it (no CPU fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "ib.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ib_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def so():
    from paper_math_0301321_b200 import _build
    return _build.build()


def test_library_exports_every_declared_symbol(so):
    names = _declared()
    assert len(names) >= 20
    lib = ctypes.CDLL(so)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    from paper_math_0301321_b200 import ib
    assert set(names) == set(ib.EXPORTS)


def test_library_is_sm100a_and_has_no_host_fallback(so):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    syms = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    assert "ibo_" not in syms          # no oracle code inside the product library


def test_binding_fails_loudly_without_library(tmp_path):
    from paper_math_0301321_b200 import ib
    saved = ib._lib
    ib._lib = None
    try:
        with pytest.raises(ImportError):
            ib.load(str(tmp_path / "missing.so"))
    finally:
        ib._lib = saved


def test_product_does_not_import_oracle():
    import subprocess, sys
    code = ("import sys; import paper_math_0301321_b200, paper_math_0301321_b200.ib; "
            "assert 'oracle' not in sys.modules, 'product imported the oracle'")
    subprocess.check_call([sys.executable, "-c", code], cwd=ROOT)
    for f in os.listdir(os.path.join(ROOT, "paper_math_0301321_b200")):
        if f.endswith((".py", ".cu", ".cuh")):
            txt = open(os.path.join(ROOT, "paper_math_0301321_b200", f)).read()
            assert "import oracle" not in txt and "ib_oracle" not in txt, f


def test_create_rejects_bad_arguments_without_gpu(so):
    # validation happens before any CUDA call
    from paper_math_0301321_b200 import ib
    L = ib.load()
    for args in ((12, 1 / 12, 1, 0.01, 1e-3), (4, 0.25, 1, 0.01, 1e-3), (16, 0.0, 1, 0.01, 1e-3),
                 (16, 1 / 16, -1, 0.01, 1e-3), (16, 1 / 16, 1, -0.1, 1e-3), (16, 1 / 16, 1, 0.01, 0)):
        assert not L.ib_create(*args)
        assert L.ib_last_error()
