"""C-ABI checks that need no GPU: the library loads, exports every symbol include/dynaspec.h
declares, and its pure host helpers / synchronous validation behave as documented."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "dynaspec.h")


def declared_functions():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dynaspec_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2510_13847_b200 import dynaspec as D
    names = declared_functions()
    assert len(names) >= 16
    lib = ctypes.CDLL(D.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(D.EXPORTED) == names


def test_budget_matches_paper_schedule():
    from paper_2510_13847_b200 import dynaspec as D
    assert [D.budget(t, 16, 1) for t in range(5)] == [16, 16, 2, 2, 1]
    assert D.budget(5, 4, 1) == 1
    assert [D.budget(t, 32, 8) for t in range(8)] == [32, 32, 8, 8, 8, 8, 8, 8]
    assert D.budget(-1, 4, 1) == -1 and D.budget(0, 4, 0) == -1 and D.budget(0, 2, 3) == -1


def test_budget_agrees_with_oracle_exhaustively():
    from oracle import dynaspec_oracle as O
    from paper_2510_13847_b200 import dynaspec as D
    for kmax in range(1, 70):
        for kmin in range(1, kmax + 1, 3):
            for t in range(0, 40):
                assert D.budget(t, kmax, kmin) == O.budget(t, kmax, kmin)


def test_pa_fr_budget_matches_paper_and_oracle():
    """K_fr(t) (App. A.1): K_max at t = 0, 1; floor(K_max / (t + 1)) after, >= 1 (R26)."""
    from oracle import dynaspec_oracle as O
    from paper_2510_13847_b200 import dynaspec as D
    assert [D.pa_fr_budget(t, 32768) for t in range(6)] == [32768, 32768, 10922, 8192, 6553, 5461]
    for K in (1, 2, 7, 1000, 32768):
        for t in range(0, 30):
            assert D.pa_fr_budget(t, K) == O.budget_pa_fr(t, K)
    assert D.lib().dynaspec_pa_fr_budget(-1, 4) == -1 and D.lib().dynaspec_pa_fr_budget(0, 0) == -1


def test_status_strings_and_sync_validation():
    from paper_2510_13847_b200 import dynaspec as D
    lib = D.lib()
    for code in range(13):
        assert lib.dynaspec_status_string(code)
    # NULL pointers / bad sizes are rejected synchronously, before any CUDA call
    c = D.DsClusters(100, 16, 4, 0, 1, 30, None, None, None, None)
    assert lib.dynaspec_head_forward(ctypes.byref(c), None, 1, None, None, None, 0, 8, 0, None, None, None, None,
                                     None, 0, None, 0, None) == 1
    assert lib.dynaspec_select(None, 1, ctypes.byref(c), 1, None, 0, None, None, None, None) == 1
    assert lib.dynaspec_layout(None, None, 0, 10, 8, 2, None, None, None, None, None, 0, None) == 1
    r = D.DsRouter(16, 0, 4, 7, ctypes.c_void_p(16), ctypes.c_void_p(16), None, None)
    assert lib.dynaspec_meta_score(ctypes.byref(r), ctypes.c_void_p(16), ctypes.c_void_p(16), 1,
                                   ctypes.c_void_p(16), None, 0, None) == 2           # dtype
    c2 = D.DsClusters(100, 12, 4, 0, 1, 30, None, ctypes.c_void_p(16), ctypes.c_void_p(16), ctypes.c_void_p(16))
    assert lib.dynaspec_head_forward(ctypes.byref(c2), ctypes.c_void_p(16), 1, ctypes.c_void_p(16),
                                     ctypes.c_void_p(16), ctypes.c_void_p(16), 0, 8, 0, ctypes.c_void_p(16),
                                     ctypes.c_void_p(16), ctypes.c_void_p(16), ctypes.c_void_p(16), None, 0,
                                     None, 0, None) == 11                              # d % 8 != 0
    c3 = D.DsClusters(100, 16, 0, 0, 1, 30, None, ctypes.c_void_p(16), ctypes.c_void_p(16), ctypes.c_void_p(16))
    assert lib.dynaspec_head_forward(ctypes.byref(c3), ctypes.c_void_p(16), 1, ctypes.c_void_p(16),
                                     ctypes.c_void_p(16), ctypes.c_void_p(16), 0, 8, 0, ctypes.c_void_p(16),
                                     ctypes.c_void_p(16), ctypes.c_void_p(16), ctypes.c_void_p(16), None, 0,
                                     None, 0, None) == 4                               # M < 1
    assert lib.dynaspec_head_forward(ctypes.byref(c2), None, 1, None, None, None, 0, 0, 0, None, None, None, None,
                                     None, 0, None, 0, None) in (1, 3, 11)
    assert lib.dynaspec_max_shortlist(ctypes.byref(c), 2) == 60
    assert lib.dynaspec_max_shortlist(ctypes.byref(c), 9) == 100


def test_kernels_are_sm100a_and_use_tma():
    """The fatbin holds sm_100a SASS with bulk-copy (TMA) instructions in the head kernel."""
    import shutil
    import subprocess
    from paper_2510_13847_b200 import dynaspec as D
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "-sass", D.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "UBLKCP" in out                 # cp.async.bulk (TMA 1D) in the head kernel
    assert "head_kernel" in out
