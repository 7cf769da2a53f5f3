import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a kernels")
    config.addinivalue_line("markers", "reference: needs /root/reference (build container only)")
    config.addinivalue_line("markers", "slow: long-running")


def _cuda_ok() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    has_gpu = _cuda_ok()
    has_ref = os.path.isdir(REFERENCE_SRC)
    skip_gpu = pytest.mark.skip(reason="no CUDA device")
    skip_ref = pytest.mark.skip(reason="/root/reference not present")
    for item in items:
        if "gpu" in item.keywords and not has_gpu:
            item.add_marker(skip_gpu)
        if "reference" in item.keywords and not has_ref:
            item.add_marker(skip_ref)


@pytest.fixture(scope="session")
def oracle():
    import oracle as orc

    orc.build()
    orc.lib()
    return orc


@pytest.fixture(scope="session")
def reference():
    """The reference package itself (build container only)."""
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    sys.dont_write_bytecode = True
    import boardbatch

    return boardbatch


@pytest.fixture(scope="session")
def reference_optional():
    if not os.path.isdir(REFERENCE_SRC):
        return None
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    sys.dont_write_bytecode = True
    import boardbatch

    return boardbatch


_TUS = ("go", "chess", "shogi", "backgammon", "small", "mcts", "fingerprint", "util")


@pytest.fixture(autouse=True)
def _checked_build(request):
    """BBK_EXPECT_CHECKED=1 (with BBK_LIB pointing at tools/checked_build.sh's library): every GPU test
    must leave the device-side scratch-index / capacity checks clean (common.cuh BBK_CHECK)."""
    if os.environ.get("BBK_EXPECT_CHECKED") != "1" or "gpu" not in request.keywords:
        yield
        return
    import ctypes

    from paper_2303_17503_b200 import _native

    L = _native.lib()
    assert L.bbk_debug_checks() == 1, "BBK_EXPECT_CHECKED=1 but the loaded library is not a checked build"
    out = (ctypes.c_ulonglong * len(_TUS))()
    L.bbk_debug_failures(1, out, len(_TUS))   # clear
    yield
    import torch

    torch.cuda.synchronize()
    bad = L.bbk_debug_failures(1, out, len(_TUS))
    fails = {t: (v >> 32, v & 0xFFFFFFFF) for t, v in zip(_TUS, out) if v}
    log = os.environ.get("BBK_CHECK_LOG")
    if log:
        with open(log, "a") as fh:
            fh.write(f"{request.node.nodeid} {'FAIL ' + repr(fails) if bad else 'clean'}\n")
    assert not bad, f"device checks failed (unit: (first line, count)): {fails}"
