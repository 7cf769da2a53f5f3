"""CLI host logic without a GPU: exit codes and the serve protocol's non-engine ops
(reference tests/test_cli.py:47-73, cli.py:33-36, 169-232)."""

import io
import json

import pytest

from paper_2303_17503_b200.cli import EXIT_UNSUPPORTED, EXIT_USAGE, _Server, main


def test_usage_error_exit_code():
    with pytest.raises(SystemExit) as exc:
        main(["bench", "--game", "tic_tac_toe"])   # missing required args
    assert exc.value.code == EXIT_USAGE
    with pytest.raises(SystemExit) as exc:
        main(["frobnicate"])
    assert exc.value.code == EXIT_USAGE
    with pytest.raises(SystemExit) as exc:
        main(["trace", "--game", "go_9x9", "--batch", "2", "--steps", "1", "--out", "x", "--format", "xml"])
    assert exc.value.code == EXIT_USAGE


def test_unsupported_game_exit_code():
    assert main(["bench", "--game", "nonsense", "--batch", "2", "--steps", "2"]) == EXIT_UNSUPPORTED
    assert main(["trace", "--game", "nonsense", "--batch", "2", "--steps", "2", "--out", "/tmp/x"]) == EXIT_UNSUPPORTED


def test_bad_agent_label_is_a_usage_error():
    assert main(["play", "--game", "tic_tac_toe", "--agents", "random,alphazero", "--games", "1"]) == EXIT_USAGE


def _run(lines):
    out = io.BytesIO()
    _Server(out).run([json.dumps(x) for x in lines])
    return [json.loads(l) for l in out.getvalue().decode().splitlines()]


def test_serve_spec_errors_and_shutdown_without_engine_calls():
    replies = _run([
        {"op": "spec", "game_id": "go_9x9"},
        {"op": "spec", "game_id": "chess"},
        {"op": "spec", "game_id": "nonsense"},
        {"op": "make", "game_id": "nonsense", "batch_size": 2, "seed": 0},
        {"op": "step", "handle": 7, "actions": [0]},
        {"op": "close", "handle": 7},
        {"op": "frobnicate"},
        {},
        {"op": "shutdown"},
        {"op": "spec", "game_id": "go_9x9"},   # after shutdown: never answered
    ])
    assert len(replies) == 9
    assert replies[0] == {"ok": True, "spec": {"game_id": "go_9x9", "num_players": 2,
                                               "observation_shape": [9, 9, 17], "num_actions": 82}}
    assert replies[1]["spec"]["num_actions"] == 4672
    assert replies[2]["ok"] is False and replies[2]["error"] == "UnsupportedGame"
    assert replies[3]["error"] == "UnsupportedGame"
    assert replies[4]["error"] == "KeyError"
    assert replies[5] == {"ok": True}
    assert replies[6]["error"] == "UsageError"
    assert replies[7]["error"] == "KeyError"
    assert replies[8] == {"ok": True}
