"""CLI ``trace`` / ``serve`` over the device path (reference cli.py:139-232).

JSON fidelity: this repo's ``trace`` writes files byte-identical to the reference's own trace
documents (sha256 fixtures made by tests/golden/make_golden_cli.py from the reference CLI), and the
``serve`` protocol replays them exactly -- in the reference's JSON form and in the binary wire form
(pack_outputs frames), port of reference tests/test_cli.py:76-126.
"""

import hashlib
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2303_17503_b200.cli import main, read_binary_trace
from paper_2303_17503_b200.session import unpack_outputs

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
GOLD = json.load(open(os.path.join(HERE, "golden", "cli_traces.json")))["traces"]


def _serve(requests, timeout=300):
    proc = subprocess.run([sys.executable, "-m", "paper_2303_17503_b200.cli", "serve"],
                          input=("\n".join(json.dumps(r) for r in requests) + "\n").encode(),
                          capture_output=True, timeout=timeout, cwd=ROOT)
    assert proc.returncode == 0, proc.stderr.decode()[-2000:]
    return proc.stdout


def _split_replies(raw: bytes):
    """JSON reply lines, each followed by `nbytes` raw bytes when it announces a binary frame."""
    out, pos = [], 0
    while pos < len(raw):
        nl = raw.index(b"\n", pos)
        rep = json.loads(raw[pos:nl])
        pos = nl + 1
        payload = None
        if "nbytes" in rep:
            payload = raw[pos:pos + rep["nbytes"]]
            pos += rep["nbytes"]
        out.append((rep, payload))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(GOLD))
def test_trace_bytes_equal_reference(name, tmp_path):
    g = GOLD[name]
    path = tmp_path / "t.json"
    assert main(["trace", "--game", g["game"], "--batch", str(g["batch"]), "--steps", str(g["steps"]),
                 "--seed", str(g["seed"]), "--out", str(path)]) == 0
    data = path.read_bytes()
    assert len(data) == g["nbytes"]
    assert hashlib.sha256(data).hexdigest() == g["sha256"]


@pytest.mark.gpu
@pytest.mark.parametrize("wire", ["json", "binary"])
def test_trace_and_serve_agree(tmp_path, wire):
    """Port of reference tests/test_cli.py:76-103, plus the same replay over binary frames."""
    path = tmp_path / "trace.json"
    assert main(["trace", "--game", "connect_four", "--batch", "3", "--steps", "15", "--seed", "9",
                 "--out", str(path)]) == 0
    doc = json.load(open(path))
    assert doc["spec"]["observation_shape"] == [6, 7, 2]
    reqs = [{"op": "make", "game_id": "connect_four", "batch_size": 3, "seed": 9, "wire": wire}]
    reqs += [{"op": "step", "handle": 1, "actions": s["actions"], "wire": wire} for s in doc["steps"]]
    reqs.append({"op": "shutdown"})
    replies = _split_replies(_serve(reqs))
    assert len(replies) == len(reqs)
    assert all(r["ok"] for r, _ in replies)

    def outputs(rep, payload):
        if wire == "json":
            return rep["outputs"]
        return {k: v.tolist() for k, v in unpack_outputs(payload).items()}

    assert outputs(*replies[0]) == doc["initial"]
    for s, (rep, payload) in zip(doc["steps"], replies[1:-1]):
        assert outputs(rep, payload) == s["outputs"]


@pytest.mark.gpu
def test_binary_trace_equals_json_trace(tmp_path):
    g = GOLD["go_9x9_b4_s40_seed1"]
    args = ["--game", "go_9x9", "--batch", "4", "--steps", "40", "--seed", "1"]
    assert main(["trace", *args, "--out", str(tmp_path / "t.json")]) == 0
    assert main(["trace", *args, "--out", str(tmp_path / "t.bin"), "--format", "binary"]) == 0
    doc = json.load(open(tmp_path / "t.json"))
    assert hashlib.sha256((tmp_path / "t.json").read_bytes()).hexdigest() == g["sha256"]
    bt = read_binary_trace(tmp_path / "t.bin")
    assert bt["header"]["spec"] == doc["spec"] and bt["header"]["steps"] == 40
    assert {k: v.tolist() for k, v in bt["initial"].items()} == doc["initial"]
    assert len(bt["steps"]) == len(doc["steps"])
    for s, b in zip(doc["steps"], bt["steps"]):
        assert b["actions"].tolist() == s["actions"]
        assert {k: v.tolist() for k, v in b["outputs"].items()} == s["outputs"]
        assert b["outputs"]["observations"].dtype == np.float32


@pytest.mark.gpu
def test_serve_random_actions_follow_the_session_schedule(tmp_path):
    """`"actions": "random"` draws the BatchSession's random actions on the device: the replies
    carry the same actions and outputs as the trace of the same seed (go_9x9 and backgammon)."""
    for game, n, steps, seed in (("go_9x9", 4, 12, 1), ("backgammon", 3, 10, 2)):
        path = tmp_path / f"{game}.json"
        assert main(["trace", "--game", game, "--batch", str(n), "--steps", str(steps), "--seed", str(seed),
                     "--out", str(path)]) == 0
        doc = json.load(open(path))
        reqs = [{"op": "make", "game_id": game, "batch_size": n, "seed": seed}]
        reqs += [{"op": "step", "handle": 1, "actions": "random", "wire": "binary"} for _ in range(steps)]
        reqs += [{"op": "observe", "handle": 1, "player": 0}, {"op": "close", "handle": 1}, {"op": "shutdown"}]
        replies = _split_replies(_serve(reqs))
        assert all(r["ok"] for r, _ in replies)
        assert replies[0][0]["outputs"] == doc["initial"]
        for s, (rep, payload) in zip(doc["steps"], replies[1:1 + steps]):
            assert rep["actions"] == s["actions"]
            assert {k: v.tolist() for k, v in unpack_outputs(payload).items()} == s["outputs"]
        obs = np.asarray(replies[1 + steps][0]["observations"])
        assert obs.shape == (n,) + tuple(doc["spec"]["observation_shape"])


@pytest.mark.gpu
def test_serve_reports_errors_and_keeps_serving():
    """Port of reference tests/test_cli.py:106-126 (chess is implemented here, so the unsupported
    game of the first request is a name the registry does not know)."""
    reqs = [
        {"op": "make", "game_id": "no_such_game", "batch_size": 2, "seed": 0},
        {"op": "make", "game_id": "kuhn_poker", "batch_size": 2, "seed": 0},
        {"op": "step", "handle": 1, "actions": [0]},
        {"op": "spec", "game_id": "go_9x9"},
        {"op": "frobnicate"},
        {"op": "step", "handle": 1, "actions": [0, 0], "wire": "xml"},
        {"op": "shutdown"},
    ]
    replies = [r for r, _ in _split_replies(_serve(reqs))]
    assert replies[0]["ok"] is False and replies[0]["error"] == "UnsupportedGame"
    assert replies[1]["ok"] is True
    assert replies[2]["ok"] is False and replies[2]["error"] == "ShapeMismatch"
    assert replies[3]["ok"] is True and replies[3]["spec"]["num_actions"] == 82
    assert replies[4]["ok"] is False and replies[4]["error"] == "UsageError"
    assert replies[5]["ok"] is False and replies[5]["error"] == "ValueError"
    assert replies[6] == {"ok": True}


@pytest.mark.gpu
def test_bench_and_play_subcommands(tmp_path, capsys):
    """Ports of reference tests/test_cli.py:12-44 through the device engines."""
    import csv

    out = tmp_path / "bench.csv"
    assert main(["bench", "--game", "tic_tac_toe", "--batch", "8", "--steps", "20", "--seed", "5",
                 "--out", str(out)]) == 0
    assert "samples/s" in capsys.readouterr().out
    assert list(csv.DictReader(open(out)))[0]["game_id"] == "tic_tac_toe"
    out = tmp_path / "long.csv"
    assert main(["bench", "--game", "hex", "--batch", "4", "--steps", "5", "--out", str(out), "--long"]) == 0
    assert {"metric", "value"} <= set(list(csv.DictReader(open(out)))[0].keys())
    out = tmp_path / "m.csv"
    assert main(["play", "--game", "tic_tac_toe", "--agents", "random,random", "--games", "10", "--seed", "1",
                 "--out", str(out)]) == 0
    rows = list(csv.DictReader(open(out)))
    assert len(rows) == 1 and int(rows[0]["wins_a"]) + int(rows[0]["wins_b"]) + int(rows[0]["draws"]) == 10
    assert main(["bench", "--game", "tic_tac_toe", "--batch", "2", "--steps", "2",
                 "--out", "/no_such_dir_abc/x.csv"]) == 4
