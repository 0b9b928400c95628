"""TEST INFRASTRUCTURE ONLY — CPU oracles for the tsgm hot path.

Two checkers live here, both loaded through ctypes:

* ``port``: ``oracle/_ref/liboracle.so``, the plain-C restatement of the
  reference algorithm (``oracle/tsgm_oracle.c``).
* ``reference``: ``oracle/_ref/libtsgm_ref.so``, the UNMODIFIED reference
  sources from /root/reference/proj/src compiled in place (``oracle/Makefile``)
  behind the C-ABI harness ``oracle/ref_runner.cpp``.

Only tests/, bench.py (cpu_baseline leg and ``--impl reference``) and
``__graft_entry__.smoke()`` may import this package, and only as the checker or
the CPU baseline. The product package never imports it.
"""
from .oracle import (  # noqa: F401
    Calib, SgmParams, FilterConfig, Port, Reference, port, reference, build,
)
