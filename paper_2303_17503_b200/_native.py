"""ctypes binding of the C-ABI in ``include/bbk.h`` (libbbk.so).

There is no fallback: if the shared object is missing (and cannot be built
because nvcc is absent) every engine call raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

_PKG = os.path.dirname(os.path.abspath(__file__))
# BBK_LIB: A/B or checked builds (made absolute: subprocesses, e.g. the reference hook-in run, may
# start in another directory)
LIB_PATH = os.path.abspath(os.environ["BBK_LIB"]) if os.environ.get("BBK_LIB") else os.path.join(_PKG, "_lib", "libbbk.so")

_lock = threading.Lock()
_lib = None


class NativeUnavailable(RuntimeError):
    """libbbk.so (the sm_100a kernels) is not built / not loadable."""


class NativeError(RuntimeError):
    """A C-ABI call returned a CUDA error code."""


P = C.c_void_p
I64 = C.c_int64
U64 = C.c_uint64
I32 = C.c_int32


class Cols(C.Structure):
    _fields_ = [("observation", P), ("legal_action_mask", P), ("rewards", P), ("terminated", P),
                ("truncated", P), ("current_player", P), ("step_count", P), ("player_to_role", P),
                ("next_actions", P), ("next_key", U64), ("episodes", P)]


class GoState(C.Structure):
    _fields_ = [("pat", P), ("hash", P), ("hist_xor", P), ("hist_len", P), ("role_to_move", P),
                ("pass_count", P)]


class GoStore(C.Structure):
    _fields_ = [("history", P), ("bloom", P), ("lab", P), ("hist_cap", I32)]


class BgState(C.Structure):
    _fields_ = [("points", P), ("misc", P)]


class ChessState(C.Structure):
    _fields_ = [("board", P), ("misc", P), ("hist", P)]


class ShogiState(C.Structure):
    _fields_ = [("board", P), ("misc", P), ("hist", P), ("hist_cap", I32)]


class MctsTree(C.Structure):
    _fields_ = [("n_search", I64), ("max_nodes", I32), ("num_actions", I32), ("mask_words", I32), ("mt", P),
                ("visits", P), ("value_sum", P), ("parent", P), ("first_child", P), ("last_child", P),
                ("next_sibling", P), ("action", P), ("role", P), ("untried", P), ("untried_count", P),
                ("next_node", P), ("leaf", P)]


ROW_COPY_MAX = 24   # BBK_ROW_COPY_MAX


class RowCopy(C.Structure):
    _fields_ = [("src", P), ("dst", P), ("row_bytes", I64), ("unit", I64)]


class RowCopySet(C.Structure):
    _fields_ = [("count", I32), ("t", RowCopy * ROW_COPY_MAX)]


def _declare(L):
    """ctypes signatures. A symbol missing from an older library build (A/B runs with BBK_LIB)
    is skipped here; tests/test_abi.py checks that the in-tree build exports all of include/bbk.h."""
    ptr = C.POINTER

    def sig(name, argtypes=None, restype=None):
        if not hasattr(L, name):
            return
        fn = getattr(L, name)
        if argtypes is not None:
            fn.argtypes = argtypes
        if restype is not None:
            fn.restype = restype

    sig("bbk_abi_version", restype=C.c_int)
    sig("bbk_build_info", restype=C.c_char_p)
    sig("bbk_fetch_async", [C.c_int, P, P, P, P, P, P, P])
    sig("bbk_debug_checks", restype=C.c_int)
    sig("bbk_debug_failures", [C.c_int, P, C.c_int], C.c_int)
    sig("bbk_go_pat_stride", [C.c_int])
    sig("bbk_go_init", [C.c_int, ptr(Cols), ptr(GoState), ptr(GoStore), I64, I64, U64, P, I32, P])
    sig("bbk_go_step", [C.c_int, C.c_double, C.c_int, ptr(Cols), ptr(GoState), ptr(Cols), ptr(GoState), ptr(GoStore),
                        P, I64, I64, U64, P, I32, P])
    sig("bbk_go_observe", [C.c_int, P, P, P, I64, P])
    sig("bbk_go_filter_words", [C.c_int])
    sig("bbk_go_rebuild_bloom", [C.c_int, ptr(GoStore), P, I64, P])
    sig("bbk_go_relabel", [C.c_int, ptr(GoStore), P, I64, P])
    sig("bbk_bg_init", [ptr(Cols), ptr(BgState), I64, I64, U64, P, I32, P])
    sig("bbk_bg_step", [ptr(Cols), ptr(BgState), ptr(Cols), ptr(BgState), P, I64, I64, U64, P, I32, P])
    sig("bbk_bg_observe", [ptr(BgState), P, P, I64, P])
    sig("bbk_random_actions", [P, I64, I32, U64, I64, P, P])
    sig("bbk_check_actions", [P, P, P, P, I64, I32, P, P])
    sig("bbk_count_finished", [P, P, I64, P, P])
    sig("bbk_latch_finished", [P, P, P, P, C.c_int, I64, P, P, P, P, P])
    for g, S in (("chess", ChessState), ("shogi", ShogiState)):
        sig(f"bbk_{g}_init", [ptr(Cols), ptr(S), I64, I64, U64, P, I32, P])
        sig(f"bbk_{g}_load", [ptr(Cols), ptr(S), P, P, I64, I64, U64, P, I32, P])
        sig(f"bbk_{g}_step", [ptr(Cols), ptr(S), ptr(Cols), ptr(S), P, I64, I64, U64, P, I32, P])
        sig(f"bbk_{g}_observe", [ptr(S), P, P, P, I64, P])
    sig("bbk_fingerprint_stride", [C.c_int, C.c_int])
    sig("bbk_go_fingerprint", [C.c_int, ptr(Cols), ptr(GoState), I64, P, I64, P, P, P])
    sig("bbk_bg_fingerprint", [ptr(Cols), ptr(BgState), I64, P, I64, P, P, P])
    sig("bbk_chess_fingerprint", [ptr(Cols), ptr(ChessState), I64, P, I64, P, P, P])
    sig("bbk_shogi_fingerprint", [ptr(Cols), ptr(ShogiState), I64, P, I64, P, P, P])
    sig("bbk_blake2b16_host", [P, I64, P])
    sig("bbk_small_fingerprint", [C.c_int, ptr(Cols), P, I64, P, I64, P, P, P])
    sig("bbk_small_init", [C.c_int, ptr(Cols), P, I64, I64, U64, P, I32, P])
    sig("bbk_small_step", [C.c_int, ptr(Cols), P, ptr(Cols), P, P, I64, I64, U64, P, I32, P])
    sig("bbk_small_observe", [C.c_int, P, P, P, P, I64, P])
    sig("bbk_mcts_seed", [ptr(MctsTree), P, P])
    sig("bbk_mcts_untried", [ptr(MctsTree), P, P, P, P, P])
    sig("bbk_mcts_select", [ptr(MctsTree), C.c_double, P, P, P, P, P, P])
    sig("bbk_mcts_rollout_actions", [ptr(MctsTree), P, P, P, P])
    sig("bbk_mcts_latch", [P, P, P, P, P, C.c_int, I64, P, P, P, P])
    sig("bbk_mcts_backup", [ptr(MctsTree), P, C.c_double, C.c_double, P])
    sig("bbk_mcts_best", [ptr(MctsTree), P, P])
    sig("bbk_copy_rows", [ptr(RowCopySet), P, P, I64, P])
    sig("bbk_mt19937_host", [U64, P, I64, P])
    return L


def lib():
    """Load libbbk.so (building it in-tree first if sources are newer and nvcc exists)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        from . import build as _build
        try:
            if not os.environ.get("BBK_LIB") and _build.needs_build():
                _build.build()
        except Exception as exc:  # nvcc missing or compile error
            if not os.path.exists(LIB_PATH):
                raise NativeUnavailable(f"libbbk.so is not built and could not be built: {exc}") from exc
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(f"{LIB_PATH} missing; run `python -m paper_2303_17503_b200.build`")
        try:
            L = C.CDLL(LIB_PATH)
        except OSError as exc:
            raise NativeUnavailable(f"cannot load {LIB_PATH}: {exc}") from exc
        _lib = _declare(L)
        return _lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        raise NativeError(f"{what} failed with cudaError {rc}")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()


def stream_handle(device=None) -> int:
    """cudaStream_t of torch's current stream on `device`, made the CUDA runtime's current device too:
    every launch goes through here, and a kernel must run on the device that owns its buffers.
    (torch's raw-stream query: no Python Stream object per launch -- the public step path's host cost.)"""
    import torch

    C_ = torch._C
    if not hasattr(C_, "_cuda_getCurrentRawStream"):   # older / newer torch: the public (slower) path
        if device is not None:
            idx = device.index if isinstance(device, torch.device) else int(device)
            if idx is not None and torch.cuda.current_device() != idx:
                torch.cuda.set_device(idx)
        return torch.cuda.current_stream(device).cuda_stream
    if device is not None:
        idx = device.index if isinstance(device, torch.device) else int(device)
        if idx is not None and C_._cuda_getDevice() != idx:
            torch.cuda.set_device(idx)
    else:
        idx = None
    if idx is None:
        idx = C_._cuda_getDevice()
    return C_._cuda_getCurrentRawStream(idx)
