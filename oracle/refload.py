"""Loaders for the reference's own compiled code (TEST INFRASTRUCTURE ONLY).

* ``load_ref_core()`` returns the reference's Cython kernel module
  (``latfft/_kernels/_core.pyx``) compiled by ``make -C oracle ref`` into
  ``oracle/_ref/``.  It travels to the GPU box with the snapshot and is what
  ``bench.py --impl reference`` times for the candidate-hashing path.
* ``import_reference()`` imports the full reference package from
  ``/root/reference/pkg/src`` with that compiled core registered first, so
  the reference runs with BACKEND == "compiled".  Only available in the build
  container (``/root/reference`` does not exist on the GPU box); used by
  ``tests/golden/make_golden.py`` to produce the committed fixtures.
"""

from __future__ import annotations

import glob
import importlib.util
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"


def ref_core_path():
    hits = sorted(glob.glob(os.path.join(HERE, "_ref", "_core*.so")))
    return hits[0] if hits else None


def load_ref_core(name="_core"):
    """The reference's compiled gather/injectivity kernels, or None."""
    path = ref_core_path()
    if path is None:
        return None
    if name in sys.modules:
        return sys.modules[name]
    spec = importlib.util.spec_from_file_location(name, path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    sys.modules[name] = mod
    return mod


def import_reference():
    """Import /root/reference's latfft with its compiled core (container only)."""
    if not os.path.isdir(REF_SRC):
        raise RuntimeError("reference sources not present (GPU box?)")
    sys.dont_write_bytecode = True  # never write into /root/reference
    if "latfft" not in sys.modules:
        if ref_core_path() is None:
            raise RuntimeError("run `make -C oracle ref` first")
        load_ref_core("latfft._kernels._core")
        sys.path.insert(0, REF_SRC)
    import latfft  # noqa: E402

    if latfft.kernel_backend != "compiled":
        raise RuntimeError("reference did not pick up the compiled core")
    return latfft
