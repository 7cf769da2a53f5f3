"""Helpers for the committed golden fixtures (tests/golden/*.json, made by make_golden.py)."""

import hashlib
import json
import os

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def names():
    """Trajectory fixtures (make_golden*.py); the search fixtures are listed by search_names(),
    the CLI trace fixture (make_golden_cli.py) is read by test_gpu_cli.py."""
    return sorted(f[:-5] for f in os.listdir(HERE)
                  if f.endswith(".json") and not f.startswith(("mcts_", "cli_")))


def search_names():
    """UCT-search decision fixtures (make_golden_mcts.py)."""
    return sorted(f[:-5] for f in os.listdir(HERE) if f.endswith(".json") and f.startswith("mcts_"))


def load(name):
    with open(os.path.join(HERE, name + ".json")) as fh:
        return json.load(fh)


def digest(b: bytes) -> str:
    return hashlib.blake2b(b, digest_size=16).hexdigest()


def game_args(rec):
    return rec["game_id"], rec["batch"], rec["seed"], rec["max_steps"]
