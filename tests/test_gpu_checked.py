"""The checked build's device-side asserts fire (tools/checked_build.sh; common.cuh BBK_CHECK).

Runs only with BBK_EXPECT_CHECKED=1 (BBK_LIB = the checked library): a Go batch whose superko
history store is declared smaller than its step count (the history tensor itself keeps its full
size, so the overflowing appends stay inside the allocation) must be reported by
bbk_debug_failures -- the same mechanism the whole GPU suite runs clean under.
"""

import ctypes
import os

import pytest

import paper_2303_17503_b200 as bb
from paper_2303_17503_b200 import _native
from paper_2303_17503_b200.core import resolve

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(os.environ.get("BBK_EXPECT_CHECKED") != "1", reason="checked build only")]


def test_history_overflow_is_reported():
    import paper_2303_17503_b200.games.go as go

    L = _native.lib()
    assert L.bbk_debug_checks() == 1
    out = (ctypes.c_ulonglong * 8)()
    L.bbk_debug_failures(1, out, 8)
    gdef = resolve("go_9x9")
    kern = gdef.batch_kernel
    key = bb.RngKey(3)
    v = kern.init(gdef, key.child(0), 4, gdef.max_steps)
    real = kern.launch_step

    def shrunk(vv, o, *args):   # launch with a 3-entry history declared over the full-size tensor
        s = o.store
        o.store = go.GoStore(s.history, s.bloom, s.lab, 3)
        try:
            real(vv, o, *args)
        finally:
            o.store = s

    kern.launch_step = shrunk
    try:
        for t in range(1, 8):
            a = kern.random_actions(v, key.child(2 * t), None)
            v = kern.step(gdef, v, a, key.child(2 * t + 1), gdef.max_steps)
    finally:
        del kern.launch_step
    import torch

    torch.cuda.synchronize()
    bad = L.bbk_debug_failures(1, out, 8)
    assert bad == 1 and out[0] != 0 and (out[0] & 0xFFFFFFFF) > 0, list(out)   # unit 0 = go.cu
    line = out[0] >> 32
    src = open(os.path.join(os.path.dirname(_native.__file__), "csrc", "go.cu")).read().splitlines()
    assert "hist_cap" in src[line - 1], (line, src[line - 1])
