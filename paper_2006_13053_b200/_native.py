"""ctypes binding of libsfftb200.so (include/sfft_b200.h).

The library is built in-tree by ``make -C paper_2006_13053_b200`` (or
``__graft_entry__.build()``).  There is no fallback: if the shared object or a
CUDA device is missing, ``lib()`` raises, and every entry point of the package
fails loudly instead of computing on the CPU.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import ParameterError

HERE = os.path.dirname(os.path.abspath(__file__))
# SFFTB_LIB_PATH: an alternative build of the same library (A/B timing of
# kernel variants on one box); the in-tree build otherwise
LIB_PATH = os.environ.get("SFFTB_LIB_PATH") or os.path.join(HERE, "_lib", "libsfftb200.so")

SFFTB_OK, SFFTB_EINVAL, SFFTB_ENOMEM, SFFTB_ECUDA = 0, 1, 2, 3

_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_int = ctypes.c_int
_dbl = ctypes.c_double
_p = ctypes.c_void_p

# name -> (restype, argtypes)
_SIGS = {
    "sfftb_version": (ctypes.c_char_p, []),
    "sfftb_last_error": (ctypes.c_char_p, []),
    "sfftb_plan_cache_clear": (_int, []),
    "sfftb_launch_count": (_i64, []),
    "sfftb_detect_gather": (_int, [_p, _i64, _i64, _p, _i64, _i64, _p, _dbl, _dbl, _int,
                                   _p, _p]),
    "sfftb_rows_injective_mod": (_int, [_p, _i64, _i64, _i64, ctypes.POINTER(_int)]),
    "sfftb_hc_count": (_int, [_int, _dbl, _p, ctypes.POINTER(_i64)]),
    "sfftb_hc_enumerate": (_int, [_int, _dbl, _p, _p, _i64]),
    "sfftb_dft_workspace_bytes": (_i64, [_i64, _i64]),
    "sfftb_dft": (_int, [_p, _i64, _p, _i64, _i64, _i64, _int, _dbl, _p, _p]),
    "sfftb_sumsq": (_int, [_p, _i64, _i64, _i64, _p, _p]),
    "sfftb_sample_detect_workspace_bytes": (_i64, [_i64, _i64]),
    "sfftb_sample_detect_dft": (_int, [_p, _i64, _i64, _i64, _u64, _i64, _dbl, _p, _p, _p, _p,
                                       _p]),
    "sfftb_sample_detect_dft_list": (_int, [_p, _p, _i64, _i64, _i64, _i64, _u64, _i64, _dbl,
                                            _p, _p, _p, _p, _p]),
    "sfftb_zero_thresholds": (_int, [_p, _i64, _i64, _i64, _p, _p]),
    "sfftb_bitmap_words": (_i64, [_i64]),
    "sfftb_nonzero_bitmap": (_int, [_p, _i64, _i64, _i64, _p, _p, _p]),
    "sfftb_hash_hits": (_int, [_p, _i64, _i64, _p, _i64, _i64, _i64, _p, _i64, _i64, _p,
                               _p, _p]),
    "sfftb_hash_tc_recomputed": (_i64, [_int]),
    "sfftb_hash_roll_recomputed": (_i64, [_int]),
    "sfftb_hash_rollf_calls": (_i64, [_int]),
    "sfftb_hash_rollf_scaled_runs": (_i64, [_int]),
    "sfftb_compact_workspace_bytes": (_i64, [_i64, _i64]),
    "sfftb_compact_mask": (_int, [_p, _i64, _i64, _p, _p, _p, _p]),
    "sfftb_medians": (_int, [_p, _i64, _p, _i64, _i64, _i64, _p, _p, _p, _i64, _p, _p]),
    "sfftb_lattice_values": (_int, [_p, _i64, _p, _i64, _i64, _p, _p, _i64, _p, _p]),
    "sfftb_topk_workspace_bytes": (_i64, [_i64, _i64]),
    "sfftb_topk": (_int, [_p, _p, _p, _i64, _i64, _dbl, _i64, _p, _p, _p, _p, _p]),
    "sfftb_topk_grid": (_int, [_p, _p, _p, _i64, _i64, _dbl, _i64, _p, _p, _p, _p, _p]),
    "sfftb_mark_indices": (_int, [_p, _p, _i64, _i64, _p, _i64, _p]),
    "sfftb_gather_rows": (_int, [_p, _i64, _p, _p, _i64, _p, _p]),
    "sfftb_pair_product": (_int, [_p, _i64, _i64, _p, _i64, _p, _p]),
    "sfftb_row_bounds": (_int, [_p, _i64, _i64, _p, _p]),
    "sfftb_anchor_coeffs": (_int, [_p, _i64, _i64, _i64, _p, _p, _i64, _p, _p]),
    "sfftb_scatter_workspace_bytes": (_i64, [_i64, _i64]),
    "sfftb_scatter_bins": (_int, [_p, _i64, _i64, _i64, _p, _p, _i64, _i64, _i64, _p, _p,
                                  _p]),
    "sfftb_scatter_list": (_int, [_p, _i64, _i64, _i64, _p, _p, _i64, _i64, _i64, _p, _p,
                                  _p]),
    "sfftb_eval_dense": (_int, [_p, _i64, _i64, _p, _p, _i64, _p, _p]),
    "sfftb_eval_lines": (_int, [_p, _i64, _i64, _p, _p, _i64, _i64, _i64, _p, _p]),
    "sfftb_add_noise": (_int, [_p, _i64, _i64, _u64, _i64, _dbl, _p]),
    "sfftb_injective_mod_dev": (_int, [_p, _i64, _i64, _i64, ctypes.POINTER(_int), _p]),
    "sfftb_sfft_stage": (_int, [_p, _p]),
    "sfftb_rows_hits_medians": (_int, [_p, _i64, _i64, _dbl, _dbl, _int, _p, _p, _p]),
    "sfftb_threshold_mask": (_int, [_p, _i64, _dbl, _p, _p]),
    "sfftb_pair_residues": (_int, [_p, _i64, _i64, _p, _i64, _p, _i64, _i64, _p, _p, _p]),
    "sfftb_hash_pairs_smem_bytes": (_i64, [_i64, _i64, _i64]),
    "sfftb_hash_pairs": (_int, [_p, _p, _i64, _i64, _i64, _i64, _i64, _p, _i64, _p, _p, _p]),
    "sfftb_medians_pairs": (_int, [_p, _p, _i64, _i64, _i64, _i64, _i64, _p, _p, _p, _i64, _p,
                                   _p]),
    "sfftb_canonicalize_workspace_bytes": (_i64, [_i64, _i64]),
    "sfftb_canonicalize_rows": (_int, [_p, _i64, _i64, _p, _p, _p, _p]),
    "sfftb_random_box_rows": (_int, [_i64, _i64, _i64, _i64, _u64, _p, _p]),
    "sfftb_r1l_workspace_bytes": (_i64, [_i64, _i64, _i64]),
    "sfftb_postprocess_r1l": (_int, [_p, _i64, _i64, _p, _p, _i64, _i64, _p, _p, _dbl, _p, _p,
                                     _p, _p]),
    "sfftb_compact_mask_cap": (_int, [_p, _i64, _i64, _i64, _p, _p, _p, _p, _p]),
    "sfftb_detect_dev_workspace_bytes": (_i64, [_i64, _i64, _i64]),
    "sfftb_detect_dev": (_int, [_p, _i64, _i64, _p, _i64, _i64, _p, _p, _i64, _i64, _int, _p, _p,
                                _p, _p, _p, _p, _p, _p]),
    "sfftb_step1_select": (_int, [_p, _i64, _i64, _p, _i64, _i64, _i64, _dbl, _p, _p, _p]),
    "sfftb_rows_in_sorted": (_int, [_p, _i64, _i64, _p, _i64, _p, _p]),
    "sfftb_alias_classify": (_int, [_p, _p, _p, _i64, _i64, _p, _dbl, _p, _p, _p]),
    "sfftb_spline_sum_lattice": (_int, [_i64, _p, _i64, _p, _p, _p, _i64, _i64, _i64, _i64, _p,
                                        _p, _p]),
    "sfftb_spline_sum_points": (_int, [_i64, _p, _i64, _p, _p, _p, _i64, _p, _p]),
    "sfftb_pcg64_seed": (_int, [_p, _i64, _i64, _p]),
    "sfftb_pcg64_random": (_int, [_p, _i64, _i64, _p]),
    "sfftb_pcg64_integers": (_int, [_p, _i64, _i64, _i64, _i64, _p]),
    "sfftb_pcg64_advance": (_int, [_p, _u64, _p]),
    "sfftb_pcg64_choice_tail": (_int, [_p, _i64, _i64, _int, _p]),
    "sfftb_box_integers_workspace_bytes": (_i64, [_i64, _i64]),
    "sfftb_box_integers": (_int, [_p, _p, _i64, _i64, _i64, _i64, _p, _p,
                                  ctypes.POINTER(_i64), ctypes.POINTER(_u64), _p]),
}

_LIB = None
_LOCK = threading.Lock()


class NativeLibraryMissing(RuntimeError):
    """libsfftb200.so is not built (run ``make -C paper_2006_13053_b200``)."""


def lib():
    global _LIB
    if _LIB is not None:
        return _LIB
    with _LOCK:
        if _LIB is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryMissing(
                    f"{LIB_PATH} is missing; build it with "
                    "`make -C paper_2006_13053_b200` (there is no CPU fallback)")
            so = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(so, name)
                fn.restype = res
                fn.argtypes = args
            _LIB = so
    return _LIB


def check(rc, what=""):
    """Map a status code to the reference's exception types."""
    if rc == SFFTB_OK:
        return
    msg = lib().sfftb_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if rc == SFFTB_EINVAL:
        raise ParameterError(msg)
    if rc == SFFTB_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


_TIMELINE = None


class Timeline:
    """Record CUDA events around every C-ABI call made while active.

    Events are recorded on the current torch stream -- the stream the
    library launches on -- so ``ms()`` gives each entry point's device time
    (used by bench.py for the per-kernel roofline numbers)."""

    def __init__(self):
        self.records = []

    def __enter__(self):
        global _TIMELINE
        self._prev, _TIMELINE = _TIMELINE, self
        return self

    def __exit__(self, *exc):
        global _TIMELINE
        _TIMELINE = self._prev
        return False

    def ms(self):
        """{entry point: [ms per call, ...]} (synchronises)."""
        import torch

        torch.cuda.synchronize()
        out = {}
        for name, a, b in self.records:
            out.setdefault(name, []).append(a.elapsed_time(b))
        return out


def call(name, *args):
    tl = _TIMELINE
    if tl is None:
        check(getattr(lib(), name)(*args), name)
        return
    import torch

    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    rc = getattr(lib(), name)(*args)
    b.record()
    tl.records.append((name, a, b))
    check(rc, name)


def launch_count():
    return int(lib().sfftb_launch_count())


def version():
    return lib().sfftb_version().decode()
