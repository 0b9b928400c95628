"""Backends the parity tests run against, behind one numpy-level API.

* ``port``: the C oracle (CPU). Not gpu-marked: it pins the oracle against the
  reference's golden vectors on every CPU run.
* ``gpu``: the product (paper_1809_07986_b200) through its C-ABI on cuda:0.
  Marked ``gpu``; fails loudly if the CUDA library is missing.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
BACKENDS = [
    pytest.param("port", id="port"),
    pytest.param("gpu", id="gpu", marks=pytest.mark.gpu),
]

_cache: dict = {}


def golden(name: str) -> dict:
    if name not in _cache:
        with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
            _cache[name] = {k: z[k] for k in z.files}
    return _cache[name]


def names(g: dict, suffix: str) -> list[str]:
    """Prefixes p such that p + suffix is a key (cases inside a group)."""
    out = []
    for k in g:
        if k.endswith(suffix):
            out.append(k[: -len(suffix)])
    return sorted(out)


def get_backend(name: str):
    if name == "port":
        from oracle import oracle as o
        if not os.path.exists(o.PORT_SO):
            o.build(reference=False)
        return o.port()
    if name == "gpu":
        from paper_1809_07986_b200.testing import GpuBackend
        return GpuBackend.shared()
    raise ValueError(name)


def backend_fixture():
    @pytest.fixture(params=BACKENDS)
    def backend(request):
        return get_backend(request.param)
    return backend
