"""CPU checks of the C ABI library: it loads without a GPU, exports every
symbol include/trstmi_b200.h declares, and its host-only pieces (seeded start
frames, schedule, Welch bound, CAS lane rule) agree with the oracle."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2207_06374_b200 import abi, api
from tests import oracle_ffi as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "trstmi_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(trstmi_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = api.load_library()
    names = declared_functions()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_struct_layouts_match_header():
    assert ctypes.sizeof(abi.Cfg) == 4 * 4 + 8 * abi.MAX_STAGES + 8 * 7 + 4 * 2 + 8 + 4 * 2
    assert ctypes.sizeof(abi.TrialOut) == 64
    assert ctypes.sizeof(abi.StageOut) == 40
    assert ctypes.sizeof(abi.OuterOut) == 64


def test_defaults_match_reference():
    lib = api.load_library()
    c = abi.Cfg()
    lib.trstmi_cfg_defaults(ctypes.byref(c), abi.COMPLEX, 2, 100)
    ref = abi.default_cfg(abi.COMPLEX, 2, 100)
    for f, _ in abi.Cfg._fields_:
        if f != "schedule":
            assert getattr(c, f) == getattr(ref, f), f
    assert (c.delta_max, c.eta, c.shrink, c.grow, c.grad_tol, c.max_outer, c.cg_force_c) == \
           (1e3, 0.05, 0.25, 2.0, 1e-9, 200, 0.5)  # trust_region.hpp:20-30


@pytest.mark.parametrize("field,d,N", [(abi.COMPLEX, 2, 100), (abi.REAL, 4, 10), (abi.COMPLEX, 6, 36),
                                       (abi.REAL, 64, 1024), (abi.COMPLEX, 1, 3)])
def test_random_frames_match_oracle(field, d, N):
    f, st = api.random_frames(field, d, N, 0, 5, 3)
    fo, sto = orc.random_frames(field, d, N, 0, 5, 3)
    assert np.array_equal(f.view(np.uint64), fo.view(np.uint64))
    assert np.array_equal(st, sto)
    assert api.lanes(field, d, N) == abi.lanes_for(field, d, N)


def test_schedule_and_welch_match_oracle():
    for N in (2, 10, 36, 100, 4096):
        assert api.default_schedule(N) == orc.schedule(N)
        for d in (1, 2, 6, 64):
            assert api.welch_bound(d, N) == orc.lib().orc_welch_bound(d, N)
    with pytest.raises(ValueError):
        api.default_schedule(1)


def test_no_device_fails_loudly():
    """Without a GPU the product refuses to run (no CPU fallback)."""
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("GPU present")
    with pytest.raises(api.CudaError):
        api.Context(0)
