"""Golden trajectories of the reference's small engines, made by running the
REFERENCE itself in the build container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_small.py [names...]

Same record format as make_golden.py (per-step batch_fingerprint, observation and action digests,
per-slot fingerprints for the first steps). Fixture names start with ``small_``; the device replays
them in tests/test_gpu_parity.py::test_device_matches_reference_golden.
"""

from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import HERE, REF, record  # noqa: E402

JOBS = [
    ("small_tic_tac_toe_s0_b64", "tic_tac_toe", 64, 0, 60, None),
    ("small_connect_four_s0_b64", "connect_four", 64, 0, 120, None),
    ("small_othello_s0_b32", "othello", 32, 0, 160, None),
    ("small_othello_s99_b16_trunc30", "othello", 16, 99, 70, 30),
    ("small_hex_s0_b32", "hex", 32, 0, 200, None),
    ("small_2048_s0_b32", "2048", 32, 0, 400, None),
    ("small_2048_s2718_b16_trunc25", "2048", 16, 2718, 80, 25),
    ("small_kuhn_poker_s0_b64", "kuhn_poker", 64, 0, 40, None),
    ("small_leduc_holdem_s0_b64", "leduc_holdem", 64, 0, 60, None),
    ("small_leduc_holdem_s99_b32", "leduc_holdem", 32, 99, 60, None),
]


def main():
    sys.path.insert(0, REF)
    only = set(sys.argv[1:])
    for name, game, n, seed, steps, max_steps in JOBS:
        if only and name not in only:
            continue
        rec = record(name, game, n, seed, steps, max_steps=max_steps, per_slot_steps=12)
        rec["generator"] = rec["generator"].replace("make_golden.py", "make_golden_small.py")
        path = os.path.join(HERE, name + ".json")
        with open(path, "w") as fh:
            json.dump(rec, fh, separators=(",", ":"))
        print(f"{name}: {rec['steps']} steps in {rec['seconds']} s -> {os.path.getsize(path)} bytes", flush=True)


if __name__ == "__main__":
    main()
