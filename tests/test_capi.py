"""CPU checks of the drop-in boundary: the product library and the oracle
libraries load, and every entry point declared in include/tsgm_b200.h is
exported (no compute calls: there is no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]*?\b(tsgm_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def product():
    from paper_1809_07986_b200 import _build
    _build.build_all()
    return ctypes.CDLL(_build.lib_path("libtsgm_b200.so"))


def test_every_declared_symbol_is_exported(product):
    names = declared("tsgm_b200.h")
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(product, n)]
    assert not missing, missing


def test_python_binding_lists_every_export():
    from paper_1809_07986_b200 import _lib
    assert sorted(_lib.EXPORTS) == declared("tsgm_b200.h")


def test_library_is_sm100a(product):
    import subprocess
    from paper_1809_07986_b200 import _build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                          _build.lib_path("libtsgm_b200.so")], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_scene_library_exports():
    from paper_1809_07986_b200 import _build
    lib = ctypes.CDLL(_build.build_scene())
    for n in declared("tsgm_scene.h"):
        assert hasattr(lib, n), n


def test_no_gpu_fails_loudly_not_silently():
    """Without a GPU, creating an engine must raise, never fall back."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1809_07986_b200 import tsgm
    cal = tsgm.StereoCalib(100.0, 20.0, 10.0, 0.5, 40, 20, 16)
    with pytest.raises(RuntimeError):
        tsgm.Engine(tsgm.EngineConfig(cal, tsgm.SgmParams(d_max=16), tsgm.FilterConfig()))


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1809_07986_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".c", ".cpp", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "liboracle" not in text and "libtsgm_ref" not in text, f
                assert not re.search(r'#include\s*[<"][^>"]*oracle', text), f
