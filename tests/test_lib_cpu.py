"""CPU-side checks of the C ABI library: it builds for sm_100a, loads, exports every symbol
include/iga.h declares, and fails loudly (no CPU fallback) when no CUDA device is present."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "iga.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(iga_[a-z_]+)\s*\(", src)))


def test_header_declares_the_four_calls():
    d = _declared()
    for f in ("iga_space_create", "iga_csr_pattern", "iga_form_residual", "iga_form_jacobian"):
        assert f in d


def test_library_exports_every_declared_symbol():
    from paper_1305_4452_b200 import build
    so = build.build()
    lib = C.CDLL(so)
    for name in _declared():
        assert hasattr(lib, name), name
    import paper_1305_4452_b200 as iga
    assert set(_declared()) <= set(iga.EXPORTS)


def test_sass_is_sm100a():
    import subprocess
    from paper_1305_4452_b200 import build
    so = build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_1305_4452_b200 as iga
    import workloads
    with pytest.raises(iga.IgaError) as ei:
        iga.Space.from_workload(workloads.make(1, n=4))
    assert ei.value.code == 6          # IGA_ERR_CUDA


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1305_4452_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "oracle.h" not in txt and "liboracle" not in txt, f
