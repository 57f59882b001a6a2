"""CPU-side checks of the drop-in boundary: the CUDA library builds for
sm_100a, loads without a GPU, and exports every entry point declared in
include/icemorph_b200.h; without a B200 every compute call fails loudly
(there is no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2107_13887_b200 import capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "icemorph_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(im_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_reference_surface():
    syms = declared_symbols()
    for s in ("im_solve_weights", "im_eval_interpolant", "im_greedy_level", "im_run_multilevel",
              "im_build_distance_index", "im_update_volume", "im_deform"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    lib = capi.load_library()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(capi.EXPORTS) <= set(declared_symbols())


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", capi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_scalar_helpers_match_reference():
    lib = capi.load_library()
    assert lib.im_eval_wendland(1, 0.5) == 0.1875
    assert lib.im_eval_basis(capi.Basis(1, 2.0), 1.0) == 0.1875
    wf = capi.WallFunctionC()
    assert lib.im_make_wall_function(5.0, 0.02, C.byref(wf)) == 0
    assert wf.support_distance == pytest.approx(0.1, rel=1e-15)
    assert lib.im_eval_wall_function(C.byref(wf), 0.05) == pytest.approx(0.5, rel=1e-12)
    assert lib.im_eval_wall_function(C.byref(wf), 0.1) == 0.0
    zero = capi.WallFunctionC(5.0, 0.0, 0)
    assert lib.im_eval_wall_function(C.byref(zero), 0.0) == 1.0
    assert lib.im_eval_wall_function(C.byref(zero), 1e-300) == 0.0


def test_no_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError):
        capi.Context(0)


def test_cpp_api_shim_exports_reference_api():
    """libicemorph_core.so implements the reference's public C++ API
    (proj/include/icemorph) over the C-ABI."""
    lib = os.path.join(ROOT, "paper_2107_13887_b200", "libicemorph_core.so")
    out = subprocess.run(["nm", "-DC", "--defined-only", lib], capture_output=True, text=True).stdout
    for sym in ("icemorph::deform(", "icemorph::update_volume(", "icemorph::build_distance_index(",
                "icemorph::run_multilevel(", "icemorph::greedy_level(", "icemorph::solve_weights(",
                "icemorph::eval_interpolant(", "icemorph::make_wall_function(",
                "icemorph::eval_wendland("):
        assert sym in out, sym
