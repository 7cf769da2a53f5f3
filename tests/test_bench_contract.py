"""bench.py's JSON-line contract pieces that do not need a GPU."""

import json
import os
import subprocess
import sys

import paper_2303_17503_b200 as bb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_every_registered_game_has_bench_constants():
    for g in bb.available_games():
        assert g in bench.B_ALG and g in bench.DEFAULT_BATCH and g in bench.STEP_KERNEL, g
        assert bench.B_ALG[g] > 0


def test_defaults_meet_the_timing_rules():
    sys_argv = sys.argv
    try:
        sys.argv = ["bench.py"]
        a = bench.parse()
    finally:
        sys.argv = sys_argv
    assert a.gpus == 1 and a.warmup >= 3 and a.steps >= 100 and a.game == "go_19x19" and a.impl == "ours"


def test_reference_arm_line_for_a_game_without_cpu_oracle():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--game", "hex"],
                         capture_output=True, text=True, timeout=300)
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and "unavailable" in line


def test_committed_traffic_summary_covers_the_bench_games():
    for g in ("go_19x19", "chess", "shogi", "backgammon", "go_9x9"):
        traffic, src = bench.ncu_traffic(g, 1 << 10)
        assert traffic and traffic > 0 and "ncu" in src
