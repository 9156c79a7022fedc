"""C-ABI checks that need no GPU: libnpcg.so loads, exports every function
include/npcg.h declares, its pure host functions behave like the reference,
and compute entry points fail loudly (no CPU fallback) when no device exists."""
import ctypes as C
import subprocess

import pytest
import torch

from paper_2511_23227_b200 import _lib as L


def test_library_exports_every_header_symbol():
    lib = L.lib()
    declared = L.header_functions()
    assert len(declared) >= 30
    nm = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True,
                        text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in nm.splitlines() if " T " in ln}
    missing = [f for f in declared if f not in exported]
    assert not missing, missing
    for f in declared:
        getattr(lib, f)  # resolvable through ctypes
    assert set(L._SIGS) <= set(declared)


def test_exports_only_c_symbols():
    nm = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True,
                        text=True, check=True).stdout
    text_syms = [ln.split()[-1] for ln in nm.splitlines() if " T " in ln]
    npcg = [s for s in text_syms if s.startswith("npcg_")]
    assert len(npcg) == len(L.header_functions())


def test_api_version_and_status_strings():
    lib = L.lib()
    assert lib.npcg_api_version() == 1
    for code, name in L.STATUS_NAMES.items():
        assert lib.npcg_status_string(code).decode() == name


@pytest.mark.parametrize("n_out,n_in,nk,axis", [(100000, 100000, 27, 3), (10, 100000, 27, 1),
                                                (100000, 5, 27, 2), (27, 27, 27, 3)])
def test_choose_sort_axis_host(n_out, n_in, nk, axis):
    # triplets.cpp:172-179 / test_triplets.cpp:273-293
    assert L.lib().npcg_choose_sort_axis(n_out, n_in, nk) == axis


def test_null_handles_are_rejected():
    lib = L.lib()
    assert lib.npcg_context_destroy(None) == 12
    assert lib.npcg_neighbors_destroy(None) == 12
    n = C.c_int64()
    assert lib.npcg_launch_count(None, C.byref(n)) == 12
    assert lib.npcg_mvmr(None, 0, None, 3, 1, 1, 1, None, 0, None, 0, None, None) == 12


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_context_creation_fails_loudly_without_gpu():
    h = C.c_void_p()
    st = L.lib().npcg_context_create(0, None, C.byref(h))
    assert st != 0 and not h.value
    from paper_2511_23227_b200 import npconv
    with pytest.raises(npconv.Error):
        npconv.Context(0)


@pytest.mark.parametrize("t,g,ci,co,seed", [(3, 1, 64, 64, 2), (3, 1, 48, 80, 5), (5, 2, 7, 3, 9)])
def test_synthetic_generators_are_the_reference_streams(ref, t, g, ci, co, seed):
    """npcg_gen_uniform_cube / npcg_gen_features / npcg_make_weights (host
    functions of the library, synthetic.hpp:12-40, tensors.hpp:142-150) give
    the unmodified reference's values bit for bit, so the bench and the drop-in
    need no oracle/ code for their inputs."""
    import numpy as np
    from paper_2511_23227_b200 import synthetic as S
    for dt in (np.float32, np.float64):
        assert np.array_equal(S.make_weights(t, g, ci, co, seed, dt), ref.make_weights(t, g, ci, co, seed, dt))
        assert np.array_equal(S.gen_features(257, g, ci, seed, dt), ref.gen_features(257, g, ci, seed, dt))
    assert np.array_equal(S.gen_uniform_cube(1000, 2.5, seed), ref.gen_uniform_cube(1000, 2.5, seed))
    assert L.lib().npcg_gen_uniform_cube(10, 0.0, 1, None) == 7  # DomainError (synthetic.cpp:14)
    assert L.lib().npcg_make_weights(2, 1, 1, 1, 1, 0, None) == 3  # even t: ShapeError
