"""The C-ABI library loads and exports every symbol include/bbk.h declares (no GPU calls)."""

import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "bbk.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bbk_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for must in ("bbk_go_init", "bbk_go_step", "bbk_bg_init", "bbk_bg_step", "bbk_random_actions",
                 "bbk_check_actions"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_2303_17503_b200 import _native

    L = _native.lib()
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    assert L.bbk_abi_version() == 6
    from paper_2303_17503_b200.games.go import GoKernel

    for n in (5, 7, 9, 11, 13, 15, 17, 19):   # host allocation == kernel row stride
        assert L.bbk_go_filter_words(n) == GoKernel(n).filter_words
    assert [L.bbk_go_filter_words(n) for n in (9, 13, 19)] == [128, 192, 320]   # bbk.h layout note
    assert L.bbk_go_filter_words(8) == -1
    # the product build carries no device-side checks (tools/checked_build.sh makes the checked one)
    if not os.environ.get("BBK_LIB"):
        assert L.bbk_debug_checks() == 0


def test_library_is_sm100a():
    from paper_2303_17503_b200 import _native

    out = os.popen(f"cuobjdump --list-elf {_native.LIB_PATH} 2>/dev/null").read()
    assert "sm_100a" in out, out
